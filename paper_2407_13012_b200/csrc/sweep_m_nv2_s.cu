// Merged-sweep instantiations (two gate passes per HBM pass): NV=2, first-pass form S.
// an A/B experiment family: compiled only with -DQSB_VARIANTS (tools/build_variant.py)
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv2_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
#ifdef QSB_VARIANTS
  return sweepk::launch_merged_f1<2, SM_MERGED, GF_FACT_S>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
}  // namespace qsb
