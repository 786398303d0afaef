// Fast-mode sweep instantiations: NV=2, shapes SH_A3 / SH_B3 (16 warps), the staggered schedule.
// an A/B experiment family: compiled only with -DQSB_VARIANTS (tools/build_variant.py)
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv2_r3t(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
#ifdef QSB_VARIANTS
  return sweepk::launch_fast<2, SH_A3, SH_B3, 1, sweepk::kStagFlags>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
}  // namespace qsb
