// Merged-sweep instantiations, NV=2, first-pass form FACT_S: the staggered schedule.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv2_t_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_merged_f1<2, SM_MERGED, GF_FACT_S, SH_A2, SH_B2, 1, true, true>(ctx, a, g);
}
}  // namespace qsb
