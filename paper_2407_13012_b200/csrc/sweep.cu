// The fused sweep kernel — the hot path of every forward and backward layer.
//
// One launch streams the whole statevector (or the bra/ket pair) through HBM once.
// A CTA owns a 2^12-amplitude tile whose 12 "local" bits map to global index bits
// (sweep "A": bits 0..11, contiguous; sweep "B": bits 0..2 for 128-byte coalescing
// plus 9 higher target bits).  Each thread keeps 2^R amplitudes per vector in
// registers; a phase is a mapping of the 12 local bits onto (5 lane bits, W warp
// bits, R register bits).  Butterflies for register bits run in registers; between
// phases the tile is re-mapped through an XOR-swizzled shared-memory exchange
// (conflict-free 16-byte accesses).  The cost phase exp(-i*gamma*C) (compact
// index -> LUT), bra creation, <bra|C|ket>, sum_j <bra|X_j|ket> and the
// expectation value are fused at load / between gates / before the store.
#include "sweep.cuh"

using namespace qsbd;

namespace qsb {
namespace {

__device__ __forceinline__ uint32_t swz(uint32_t x) {
  return x ^ (((x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12)) & 7u);
}

__device__ __forceinline__ uint64_t tile_base(const SweepArgs& a, uint64_t tile) {
  uint64_t base = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (r < a.nruns) {
      base |= (tile & ((1ull << a.run_len[r]) - 1ull)) << a.run_pos[r];
      tile >>= a.run_len[r];
    }
  }
  return base;
}

template <int W>
__device__ __forceinline__ void thread_part(const PhaseMap& P, int lane, int warp, uint32_t& lb, uint64_t& gb) {
  lb = 0;
  gb = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    uint32_t bit = (lane >> b) & 1u;
    lb |= bit << P.lane_l[b];
    gb |= (uint64_t)bit << P.lane_g[b];
  }
#pragma unroll
  for (int b = 0; b < W; ++b) {
    uint32_t bit = (warp >> b) & 1u;
    lb |= bit << P.warp_l[b];
    gb |= (uint64_t)bit << P.warp_g[b];
  }
}

template <bool EXACT>
__device__ __forceinline__ void butterfly(double2& t, double2& u, int form, double ga, double gb) {
  if constexpr (EXACT) {
    const double c = ga, s = gb;
    double2 n0 = make_double2(__dadd_rn(__dmul_rn(c, t.x), __dmul_rn(s, u.y)),
                              __dadd_rn(__dmul_rn(c, t.y), -__dmul_rn(s, u.x)));
    double2 n1 = make_double2(__dadd_rn(__dmul_rn(s, t.y), __dmul_rn(c, u.x)),
                              __dadd_rn(__dmul_rn(c, u.y), -__dmul_rn(s, t.x)));
    t = n0;
    u = n1;
  } else {
    if (form == GF_FACT_C) {  // a = 1, b = tau
      double2 n0 = make_double2(fma(gb, u.y, t.x), fma(-gb, u.x, t.y));
      double2 n1 = make_double2(fma(gb, t.y, u.x), fma(-gb, t.x, u.y));
      t = n0;
      u = n1;
    } else {  // a = rho, b = 1
      double2 n0 = make_double2(fma(ga, t.x, u.y), fma(ga, t.y, -u.x));
      double2 n1 = make_double2(fma(ga, u.x, t.y), fma(ga, u.y, -t.x));
      t = n0;
      u = n1;
    }
  }
}

template <bool EXACT>
__device__ __forceinline__ double tval(const SweepArgs& a, uint64_t g) {
  if (a.kind == 1) return a.vmin + (double)((const uint8_t*)a.cidx)[g];
  if (a.kind == 2) return a.vmin + (double)((const uint16_t*)a.cidx)[g];
  return a.table[g];
}

template <bool EXACT>
__device__ __forceinline__ double2 phase_factor(const SweepArgs& a, const double2* slut, uint64_t g) {
  if (a.kind == 1) return slut[((const uint8_t*)a.cidx)[g]];
  if (a.kind == 2) return __ldg(&a.lut[((const uint16_t*)a.cidx)[g]]);
  double ang = a.pre_ang * a.table[g];
  double s, c;
  sincos(ang, &s, &c);
  double2 f = make_double2(c, s);
  if (!EXACT) f = cmul_fast(f, a.pre_extra);
  return f;
}

template <int R, int W, int NV, bool EXACT>
__global__ void __launch_bounds__(32 << W, (NV == 1) ? 2 : 1) k_sweep(const SweepArgs a) {
  constexpr int T = 5 + W + R;
  constexpr int NR = 1 << R;
  constexpr uint32_t TILE = 1u << T;
  static_assert(T == kSweepT, "tile size");
  extern __shared__ double2 smem[];
  double2* slut = smem + NV * TILE;  // u8 LUT (<= 256 entries)

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t flags = a.flags;

  if (a.kind == 1 && (flags & SF_PRE_PHASE)) {
    for (int i = threadIdx.x; i < a.nlut; i += blockDim.x) slut[i] = a.lut[i];
    __syncthreads();
  }

  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  double2 v[NV][NR];

  for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const uint64_t base = tile_base(a, tile);
    uint32_t lb;
    uint64_t gb;
    thread_part<W>(a.ph[0], lane, warp, lb, gb);
    int rl = a.ph[0].reg_l, rg = a.ph[0].reg_g;
    const uint64_t g0 = base + gb;

    // ---------------------------------------------------------------- load
    if (flags & SF_PLUS) {
#pragma unroll
      for (int j = 0; j < NR; ++j) v[0][j] = make_double2(a.plus_amp, 0.0);
    } else {
#pragma unroll
      for (int j = 0; j < NR; ++j) v[0][j] = ld_stream(a.v0 + g0 + ((uint64_t)j << rg));
    }
    if constexpr (NV == 2) {
      if (!(flags & SF_BRA_FROM_KET)) {
#pragma unroll
        for (int j = 0; j < NR; ++j) v[1][j] = ld_stream(a.v1 + g0 + ((uint64_t)j << rg));
      }
    }

    // ---------------------------------------------------------------- pre ops
    if (flags & (SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER)) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const uint64_t g = g0 + ((uint64_t)j << rg);
        if constexpr (NV == 2) {
          if (flags & (SF_BRA_FROM_KET | SF_PRE_DINNER)) {
            const double t = tval<EXACT>(a, g);
            if (flags & SF_BRA_FROM_KET) v[1][j] = make_double2(t * v[0][j].x, t * v[0][j].y);
            if (flags & SF_PRE_DINNER) acc1 = fma(t, v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x, acc1);
          }
        }
        if (flags & SF_PRE_PHASE) {
          const double2 f = phase_factor<EXACT>(a, slut, g);
#pragma unroll
          for (int q = 0; q < NV; ++q) v[q][j] = cmul<EXACT>(v[q][j], f);
        }
      }
    }

    // ---------------------------------------------------------------- phases
#pragma unroll 1
    for (int p = 0; p < a.nphase; ++p) {
      if (p > 0) {
        // exchange: write under the previous mapping, read under the new one
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
          for (int j = 0; j < NR; ++j) smem[q * TILE + swz(lb | ((uint32_t)j << rl))] = v[q][j];
        __syncthreads();
        thread_part<W>(a.ph[p], lane, warp, lb, gb);
        rl = a.ph[p].reg_l;
        rg = a.ph[p].reg_g;
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
          for (int j = 0; j < NR; ++j) v[q][j] = smem[q * TILE + swz(lb | ((uint32_t)j << rl))];
      }
      const uint32_t apply = a.ph[p].apply;
      double xs = 0.0;
#pragma unroll
      for (int b = 0; b < R; ++b) {
        if (apply & (1u << b)) {
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            if (j & (1 << b)) continue;
            const int k = j | (1 << b);
            if constexpr (NV == 2) {
              if (flags & SF_XSUM) {
                // Im(conj(b_j) k_k) + Im(conj(b_k) k_j)
                xs += v[1][j].x * v[0][k].y - v[1][j].y * v[0][k].x;
                xs += v[1][k].x * v[0][j].y - v[1][k].y * v[0][j].x;
              }
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) butterfly<EXACT>(v[q][j], v[q][k], a.form, a.ga, a.gb);
          }
        }
      }
      if constexpr (NV == 2) acc2 = fma(a.xs_w[p], xs, acc2);
    }

    // ---------------------------------------------------------------- post
    if (flags & SF_POST_SCALE) {
      const double sc = a.post_scale;
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int j = 0; j < NR; ++j) v[q][j] = make_double2(v[q][j].x * sc, v[q][j].y * sc);
    }
    const uint64_t g1 = base + gb;
    if (flags & (SF_POST_EXPECT | SF_POST_DINNER)) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const uint64_t g = g1 + ((uint64_t)j << rg);
        const double t = tval<EXACT>(a, g);
        if constexpr (NV == 1) {
          acc0 = fma(t, fma(v[0][j].x, v[0][j].x, v[0][j].y * v[0][j].y), acc0);
        } else {
          acc1 = fma(t, v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x, acc1);
        }
      }
    }
    if (!(flags & SF_NO_STORE)) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        double2* dst = q == 0 ? a.v0 : a.v1;
#pragma unroll
        for (int j = 0; j < NR; ++j) st_stream(dst + g1 + ((uint64_t)j << rg), v[q][j]);
      }
    }
  }

  // ------------------------------------------------------------ partial sums
  if (a.partials) {
    __syncthreads();
    double* red = (double*)smem;
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    acc2 = warp_sum(acc2);
    constexpr int NW = 1 << W;
    if (lane == 0) {
      red[warp] = acc0;
      red[NW + warp] = acc1;
      red[2 * NW + warp] = acc2;
    }
    __syncthreads();
    if (threadIdx.x < kSlots) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[threadIdx.x * NW + w];
      a.partials[threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
  }
}

template <int R, int W, int NV, bool EXACT>
struct SweepKernel {
  static constexpr int threads = 32 << W;
  static constexpr size_t smem = (size_t)NV * (1u << kSweepT) * sizeof(double2) + 256 * sizeof(double2);
  static int grid(qsb_ctx* ctx, uint64_t ntiles, unsigned* g) {
    static int occ = -1;  // per process; one device type
    if (occ < 0) {
      QSB_CUDA(cudaFuncSetAttribute(k_sweep<R, W, NV, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int o = 0;
      QSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep<R, W, NV, EXACT>, threads, smem));
      occ = o < 1 ? 1 : o;
    }
    uint64_t want = (uint64_t)ctx->num_sms * occ;
    *g = (unsigned)(ntiles < want ? ntiles : want);
    return QSB_OK;
  }
  static int launch(qsb_ctx* ctx, SweepArgs& a, unsigned* gout) {
    unsigned g;
    QSB_TRY(grid(ctx, a.ntiles, &g));
    k_sweep<R, W, NV, EXACT><<<g, threads, smem, ctx->stream>>>(a);
    QSB_CHECK_LAUNCH(ctx, "sweep");
    if (gout) *gout = g;
    return QSB_OK;
  }
};

}  // namespace

int sweep_grid(qsb_ctx* ctx, int nv, bool exact, uint64_t ntiles, unsigned* g) {
  if (nv == 1) return exact ? SweepKernel<5, 2, 1, true>::grid(ctx, ntiles, g) : SweepKernel<5, 2, 1, false>::grid(ctx, ntiles, g);
  return exact ? SweepKernel<4, 3, 2, true>::grid(ctx, ntiles, g) : SweepKernel<4, 3, 2, false>::grid(ctx, ntiles, g);
}

int launch_sweep(qsb_ctx* ctx, int nv, bool exact, SweepArgs& a, unsigned* gout) {
  if (nv == 1) return exact ? SweepKernel<5, 2, 1, true>::launch(ctx, a, gout) : SweepKernel<5, 2, 1, false>::launch(ctx, a, gout);
  return exact ? SweepKernel<4, 3, 2, true>::launch(ctx, a, gout) : SweepKernel<4, 3, 2, false>::launch(ctx, a, gout);
}

}  // namespace qsb
