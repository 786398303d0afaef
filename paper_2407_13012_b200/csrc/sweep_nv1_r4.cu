// Fast-mode sweep instantiations: NV=1, shapes SH_A2 / SH_B2 (see sweep_impl.cuh).
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv1_r4(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_fast<1, SH_A2, SH_B2, 1, 0xffffffffu, true>(ctx, a, g);
}
}  // namespace qsb
