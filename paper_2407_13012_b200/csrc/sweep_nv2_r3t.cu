// Fast-mode sweep instantiations: NV=2, shapes SH_A3 / SH_B3 (16 warps), the staggered schedule.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv2_r3t(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_fast<2, SH_A3, SH_B3, 1, sweepk::kStagFlags>(ctx, a, g);
}
}  // namespace qsb
