// Merged-sweep instantiations (two gate passes per HBM pass): NV=1, R=5 family, first-pass form C.
// an A/B experiment family: compiled only with -DQSB_VARIANTS (tools/build_variant.py)
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv1_r5_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
#ifdef QSB_VARIANTS
  return sweepk::launch_merged_f1<1, SM_MERGED, GF_FACT_C, SH_A1, SH_B1>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
}  // namespace qsb
