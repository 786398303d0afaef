// Fast-mode sweep instantiations: NV=1, shapes SH_A1 / SH_B1 (32 amplitudes per
// thread), two independent warp groups per CTA (see sweep_impl.cuh).
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_nv1_r5g(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::launch_fast<1, SH_A1, SH_B1, 2, 0xffffffffu, true>(ctx, a, g);
}
}  // namespace qsb
