// Bra/ket sweep instantiations (the adjoint walk).
#include "sweep_impl.cuh"

namespace qsb {

int launch_sweep_nv2(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::dispatch_nv<2, SH_A2, SH_A2X, SH_B2>(a, [&](auto k) { return decltype(k)::launch(ctx, a, g); });
}

int grid_sweep_nv2(qsb_ctx* ctx, SweepArgs& a, uint64_t ntiles, unsigned* g) {
  return sweepk::dispatch_nv<2, SH_A2, SH_A2X, SH_B2>(a, [&](auto k) { return decltype(k)::grid(ctx, ntiles, g); });
}

}  // namespace qsb
