// Exact-mode sweep instantiations (FMA-free, ascending qubit order; shapes A2X / B2).
#include "sweep_impl.cuh"

namespace qsb {
int launch_sweep_exact_nv1(qsb_ctx* ctx, SweepArgs& a, unsigned* g) { return sweepk::launch_exact<1>(ctx, a, g); }
int launch_sweep_exact_nv2(qsb_ctx* ctx, SweepArgs& a, unsigned* g) { return sweepk::launch_exact<2>(ctx, a, g); }
}  // namespace qsb
