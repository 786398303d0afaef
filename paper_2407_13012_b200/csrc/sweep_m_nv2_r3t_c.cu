// Merged-sweep instantiations, NV=2, R=3 shapes (16 warps), first-pass form FACT_C: the staggered schedule.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv2_r3t_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_merged_f1<2, SM_MERGED, GF_FACT_C, SH_A3, SH_B3, 1, true>(ctx, a, g);
}
}  // namespace qsb
