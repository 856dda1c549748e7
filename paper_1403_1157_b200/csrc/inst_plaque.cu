// Kernel instantiations for the plaque model (compiled as its own unit).
#include "ctx.cuh"

namespace tdg {
bool pick_plaque(int dim, int order, Impl* out) { return pick_order<PlaqueDev>(dim, order, out); }
}  // namespace tdg
