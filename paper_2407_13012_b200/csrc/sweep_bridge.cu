// Bridge-sweep instantiations: the last forward layer's window pass on the ket, <C>,
// bra = C*ket, then the first backward layer's pass on both (NV=2).
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_bridge(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {  // lock-step: an A/B family
#ifdef QSB_VARIANTS
  if (a.form == GF_FACT_C) return sweepk::launch_merged_f1<2, SM_BRIDGE, GF_FACT_C>(ctx, a, g);
  return sweepk::launch_merged_f1<2, SM_BRIDGE, GF_FACT_S>(ctx, a, g);
#else
  (void)ctx;
  (void)a;
  (void)g;
  return variant_missing();
#endif
}
// second pass staggered (see the kernel)
int launch_sweep_bridge_t(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  if (a.form == GF_FACT_C) return sweepk::launch_merged_f1<2, SM_BRIDGE, GF_FACT_C, SH_A2, SH_B2, 1, true, true>(ctx, a, g);
  return sweepk::launch_merged_f1<2, SM_BRIDGE, GF_FACT_S, SH_A2, SH_B2, 1, true, true>(ctx, a, g);
}
}  // namespace qsb
