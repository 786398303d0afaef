// Merged-sweep instantiations: NV=2, R=3 family (16 warps, 8 amplitudes per vector per
// thread), first-pass form S.
// an A/B experiment family: compiled only with -DQSB_VARIANTS (tools/build_variant.py)
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_m_nv2_r3_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
#ifdef QSB_VARIANTS
  return sweepk::launch_merged_f1<2, SM_MERGED, GF_FACT_S, SH_A3, SH_B3>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
}  // namespace qsb
