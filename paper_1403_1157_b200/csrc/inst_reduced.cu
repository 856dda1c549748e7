// Kernel instantiations for the reduced model (compiled as its own unit).
#include "ctx.cuh"

namespace tdg {
bool pick_reduced(int dim, int order, Impl* out) { return pick_order<ReducedDev>(dim, order, out); }
}  // namespace tdg
