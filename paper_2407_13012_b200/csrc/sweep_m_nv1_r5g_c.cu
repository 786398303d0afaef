// Merged-sweep instantiations: NV=1, R=5 family with two warp groups, first-pass form C.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv1_r5g_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_merged_f1<1, SM_MERGED, GF_FACT_C, SH_A1, SH_B1, 2>(ctx, a, g);
}
}  // namespace qsb
