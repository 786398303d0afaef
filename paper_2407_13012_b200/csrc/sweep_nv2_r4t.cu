// Fast-mode sweep instantiations: NV=2, shapes SH_A2 / SH_B2, the staggered schedule.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv2_r4t(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_fast<2, SH_A2, SH_B2, 1, sweepk::kStagFlags, true>(ctx, a, g);
}
}  // namespace qsb
