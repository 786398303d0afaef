// Fast-mode sweep instantiations: NV=1, shapes SH_A3 / SH_B3 (see sweep_impl.cuh).
// an A/B experiment family: compiled only with -DQSB_VARIANTS (tools/build_variant.py)
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv1_r3(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
#ifdef QSB_VARIANTS
  return sweepk::launch_fast<1, SH_A3, SH_B3>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
}  // namespace qsb
