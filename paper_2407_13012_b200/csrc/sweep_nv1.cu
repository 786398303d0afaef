// Single-vector sweep instantiations (forward layers, Rx layers).
#include "sweep_impl.cuh"

namespace qsb {

int launch_sweep_nv1(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  return sweepk::dispatch_nv<1, SH_A1, SH_A1X, SH_B1>(a, [&](auto k) { return decltype(k)::launch(ctx, a, g); });
}

int grid_sweep_nv1(qsb_ctx* ctx, SweepArgs& a, uint64_t ntiles, unsigned* g) {
  return sweepk::dispatch_nv<1, SH_A1, SH_A1X, SH_B1>(a, [&](auto k) { return decltype(k)::grid(ctx, ntiles, g); });
}

}  // namespace qsb
