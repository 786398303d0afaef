// Merged-sweep instantiations (two gate passes per HBM pass): NV=1, R=4 family, first-pass form C.
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv1_r4_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_merged_f1<1, SM_MERGED, GF_FACT_C, SH_A2, SH_B2, 1, false, true>(ctx, a, g);
}
}  // namespace qsb
