// Kernel instantiations for the diffusion model (compiled as its own unit).
#include "ctx.cuh"

namespace tdg {
bool pick_diffusion(int dim, int order, Impl* out) { return pick_order<DiffusionDev<1>>(dim, order, out); }
}  // namespace tdg
