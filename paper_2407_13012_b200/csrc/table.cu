// Cost-table precompute (costpoly.precompute, costpoly.py:126-133 ->
// numba_impl.precompute_table :229-238) and the compact index / phase LUT used
// by the fused sweeps.
//
// T[x] = sum over terms k in the given order of w_k * [x & m_k == m_k], from 0.0.
// One thread per 4 consecutive x (32-byte stores); a warp covers 128 consecutive
// x, so a term whose mask has a bit >= 7 that is clear in the warp's common high
// bits cannot match any x of the warp and is skipped warp-uniformly.  Skipping a
// non-matching term is exactly what the reference does, so the sum is bit-exact
// for any weights.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <unordered_map>
#include <vector>

#include "common.cuh"

using namespace qsb;

namespace {

constexpr int kPreThreads = 256;
constexpr int kPreX = 4;            // x values per thread
constexpr int kTermChunk = 2048;    // terms staged in shared memory per pass

// Shard index map (sharded statevectors): local index i -> global assignment
// x = (i & (2^b - 1)) | (rank << s1) | ((i >> b) << s2).  Identity: b = 63, rank = 0.
struct IndexMap {
  uint32_t b, s1, s2;
  uint64_t rank;
  __host__ __device__ uint64_t operator()(uint64_t i) const {
    const uint64_t lo = b >= 63 ? i : (i & ((1ull << b) - 1ull));
    const uint64_t hi = b >= 63 ? 0 : ((i >> b) << s2);
    return lo | (rank << s1) | hi;
  }
};

__global__ void __launch_bounds__(kPreThreads) k_precompute(const double* __restrict__ w, const uint64_t* __restrict__ m,
                                                            uint64_t num_terms, double* __restrict__ out, uint64_t len,
                                                            IndexMap map) {
  __shared__ double sw[kTermChunk];
  __shared__ uint64_t sm[kTermChunk];
  const uint64_t i0 = ((uint64_t)blockIdx.x * kPreThreads + threadIdx.x) * kPreX;
  // the 4 indices of a thread (and the 128 of a warp, when b >= 7) map to consecutive x
  const uint64_t x0 = map(i0);
  // warp-common high bits (bits >= 7 are equal for all x of this warp)
  const bool skip_ok = map.b >= 7;
  const uint64_t warp_x = x0 & ~127ull;
  double acc[kPreX];
#pragma unroll
  for (int e = 0; e < kPreX; ++e) acc[e] = 0.0;
  for (uint64_t c0 = 0; c0 < num_terms; c0 += kTermChunk) {
    const int cn = (int)((num_terms - c0) < (uint64_t)kTermChunk ? (num_terms - c0) : kTermChunk);
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += kPreThreads) {
      sw[i] = w[c0 + i];
      sm[i] = m[c0 + i];
    }
    __syncthreads();
    for (int k = 0; k < cn; ++k) {
      const uint64_t mk = sm[k];
      if (skip_ok && ((mk & ~127ull) & ~warp_x)) continue;  // warp-uniform: no x in this warp matches
      const double wk = sw[k];
#pragma unroll
      for (int e = 0; e < kPreX; ++e)
        if (((x0 + e) & mk) == mk) acc[e] = __dadd_rn(acc[e], wk);
    }
  }
  if (i0 + kPreX <= len) {
    double2* o = (double2*)(out + i0);
    o[0] = make_double2(acc[0], acc[1]);
    o[1] = make_double2(acc[2], acc[3]);
  } else {
    for (int e = 0; e < kPreX; ++e)
      if (i0 + e < len) out[i0 + e] = acc[e];
  }
}

// ---------------------------------------------------------------- dyadic-weight path
// When every weight is a multiple of 2^-s and sum |w| * 2^s < 2^52, every partial sum
// of the reference's term-ordered loop is a multiple of 2^-s below 2^(52-s) in
// magnitude -- exactly representable -- so each addition is exact and T[x] is the
// exact sum of the matching weights, whatever the order.  (Integer weights -- every
// MaxCut / weighted MaxCut -- are the case s = 0.)  That sum is then computed in int64
// tile by tile: a tile is 4096 consecutive x sharing their high bits xh; a term with
// mask m contributes to the tile iff (m & ~0xFFF) is inside xh, and then to every x
// whose low 12 bits contain m & 0xFFF.  So W[l] = sum of those terms' weights with
// m & 0xFFF == l, and T[xh | x] = sum over l subset of x of W[l]: a subset-sum (zeta)
// transform over 12 bits -- 12 adds per x instead of one mask test per term.
// The bit-exact equality with the term-ordered double sum is what the tests check.
constexpr int kZT = 12;                 // tile bits
constexpr int kZThreads = 256;          // 16 entries per thread
constexpr uint32_t kZN = 1u << kZT;

// shared-memory word of entry x: bits 4..7 XORed into bits 0..3, so each of the three
// register maps below reads/writes 16 consecutive words per half-warp (conflict-free)
__device__ __forceinline__ uint32_t zswz(uint32_t x) { return x ^ ((x >> 4) & 15u); }

// zeta over the 4 register bits of v (v[r] += v[r without bit b] for every set bit b)
__device__ __forceinline__ void zeta_regs(long long (&v)[16]) {
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r & (1 << b)) v[r] += v[r ^ (1 << b)];
}

__global__ void __launch_bounds__(kZThreads, 4) k_precompute_zeta(const long long* __restrict__ w,
                                                               const uint64_t* __restrict__ m, uint64_t num_terms,
                                                               double* __restrict__ out, uint64_t ntiles, double scale,
                                                               IndexMap map, long long* __restrict__ minmax) {
  __shared__ long long S[kZN];
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  long long vlo = LLONG_MAX, vhi = LLONG_MIN;  // the table's min / max (int64, fused)
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t i0 = tile << kZT;
    const uint64_t xh = map(i0);  // the tile's high bits (the map is the identity on bits < 12)
#pragma unroll
    for (int r = 0; r < 16; ++r) S[tid + 256u * r] = 0;
    __syncthreads();
    // scatter the tile's terms; those with no low bits (the common case for high
    // qubits) are summed in registers and added once per warp
    long long c0 = 0;
    for (uint64_t k = tid; k < num_terms; k += kZThreads) {
      const uint64_t mk = __ldg(&m[k]);
      if ((mk & ~(uint64_t)(kZN - 1u)) & ~xh) continue;  // a high bit the tile lacks
      const uint32_t lo = (uint32_t)(mk & (kZN - 1u));
      const long long wk = __ldg(&w[k]);
      if (lo == 0) c0 += wk;
      else atomicAdd((unsigned long long*)&S[zswz(lo)], (unsigned long long)wk);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    if (lane == 0 && c0) atomicAdd((unsigned long long*)&S[0], (unsigned long long)c0);
    __syncthreads();
    long long v[16];
    // map 3: registers = bits 0..3, lanes = bits 4..8, warps = bits 9..11
    {
      const uint32_t base = tid << 4;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = S[zswz(base | r)];
      zeta_regs(v);
#pragma unroll
      for (int r = 0; r < 16; ++r) S[zswz(base | r)] = v[r];
    }
    __syncthreads();
    // map 2: registers = bits 4..7, lanes = bits 0..3 and 8, warps = bits 9..11
    {
      const uint32_t base = (tid & 15u) | ((tid >> 4) << 8);
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = S[zswz(base | (r << 4))];
      zeta_regs(v);
#pragma unroll
      for (int r = 0; r < 16; ++r) S[zswz(base | (r << 4))] = v[r];
    }
    __syncthreads();
    // map 1: registers = bits 8..11, threads = bits 0..7 -> coalesced stores
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = S[zswz(tid | (r << 8))];
    zeta_regs(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      __stcs(out + i0 + tid + 256u * r, (double)v[r] * scale);
      vlo = min(vlo, v[r]);
      vhi = max(vhi, v[r]);
    }
    __syncthreads();  // S is zeroed for the next tile
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vlo = min(vlo, __shfl_xor_sync(0xffffffffu, vlo, o));
    vhi = max(vhi, __shfl_xor_sync(0xffffffffu, vhi, o));
  }
  if (lane == 0) {
    atomicMin(&minmax[0], vlo);
    atomicMax(&minmax[1], vhi);
  }
}

__global__ void k_minmax_init(long long* mm) {
  mm[0] = LLONG_MAX;
  mm[1] = LLONG_MIN;
}

// Exact flip symmetry of a table given by merged integer terms W_m (T(x) = sum of W_m over
// m subset of x): T(~x) = sum_m W_m prod_{i in m} (1 - x_i) has the subset-basis
// coefficients D_s = (-1)^|s| sum_{m superset of s} W_m, and the basis is unique, so
// T(x) == T(~x) for every x iff D == W.  The tables of this path are exact integer sums,
// so this equals the device check values[x] == values[len-1-x] bit for bit.
// Returns 1 / 0, or -1 when the subset enumeration would be too large.
static int dyadic_symmetric(const std::vector<uint64_t>& im, const std::vector<long long>& iw) {
  uint64_t work = 0;
  for (uint64_t m : im) {
    const int d = __builtin_popcountll(m);
    if (d > 20) return -1;
    work += 1ull << d;
    if (work > (1ull << 22)) return -1;
  }
  std::unordered_map<uint64_t, long long> D;
  D.reserve(work * 2);
  for (size_t k = 0; k < im.size(); ++k) {
    const uint64_t m = im[k];
    for (uint64_t sub = m;; sub = (sub - 1) & m) {  // every subset of m
      D[sub] += (__builtin_popcountll(sub) & 1) ? -iw[k] : iw[k];
      if (!sub) break;
    }
  }
  std::unordered_map<uint64_t, long long> W;
  for (size_t k = 0; k < im.size(); ++k) W[im[k]] = iw[k];  // masks are unique here
  for (const auto& [sub, c] : D)
    if (c != 0 && (W.count(sub) ? W[sub] : 0) != c) return 0;
  for (const auto& [m, c] : W)
    if ((D.count(m) ? D[m] : 0) != c) return 0;
  return 1;
}

// the dyadic scale s of the weights (see above), or -1 when the path does not apply
static int dyadic_shift(const double* w, uint64_t num_terms) {
  for (int sh = 0; sh <= 24; ++sh) {
    double tot = 0.0;
    bool ok = true;
    for (uint64_t k = 0; k < num_terms && ok; ++k) {
      const double x = ldexp(w[k], sh);
      ok = std::isfinite(x) && x == rint(x);
      tot += fabs(x);
    }
    if (ok) return tot < 4503599627370496.0 ? sh : -1;  // 2^52 (tot itself rounds up at worst)
  }
  return -1;
}

// ---------------------------------------------------------------- float-weight path
// Any weights: the reference's term-ordered sum, per x, from 0.0.  Tiles of 4096 x
// sharing their high bits xh: the CTA compacts, in term order, the terms whose high mask
// bits lie in xh (the others cannot match any x of the tile -- the reference skips them
// too) into shared memory as (low mask, weight); each thread then runs that list over its
// 16 x with a 32-bit mask test and a predicated add.  Same additions in the same order:
// bit-exact for any weights.
constexpr int kFChunk = 2048;  // compacted terms per pass

__global__ void __launch_bounds__(kZThreads) k_precompute_tiled(const double* __restrict__ w,
                                                                const uint64_t* __restrict__ m, uint64_t num_terms,
                                                                double* __restrict__ out, uint64_t ntiles,
                                                                IndexMap map) {
  __shared__ double lw[kFChunk];
  __shared__ uint32_t lm[kFChunk];
  __shared__ uint32_t wcount[kZThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t i0 = tile << kZT;
    const uint64_t xh = map(i0);
    double acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0.0;
    const uint32_t xl = tid;  // this thread's x: xh | tid + 256 r
    uint64_t k0 = 0;
    while (k0 < num_terms) {
      // ordered compaction of the next terms until the list is full or the terms end
      uint32_t cnt = 0;
      __syncthreads();  // the previous list has been consumed
      while (k0 < num_terms && cnt + kZThreads <= (uint32_t)kFChunk) {
        const uint64_t k = k0 + tid;
        bool keep = false;
        uint64_t mk = 0;
        double wk = 0.0;
        if (k < num_terms) {
          mk = __ldg(&m[k]);
          keep = ((mk & ~(uint64_t)(kZN - 1u)) & ~xh) == 0;
          if (keep) wk = __ldg(&w[k]);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wcount[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = cnt, total = cnt;
#pragma unroll
        for (int q = 0; q < kZThreads / 32; ++q) {
          const uint32_t c = wcount[q];
          if (q < (int)warp) before += c;
          total += c;
        }
        if (keep) {
          const uint32_t pos = before + __popc(bal & ((1u << lane) - 1u));
          lm[pos] = (uint32_t)(mk & (kZN - 1u));
          lw[pos] = wk;
        }
        cnt = total;
        k0 += kZThreads;
        __syncthreads();  // wcount reuse / the list is complete
      }
      for (uint32_t j = 0; j < cnt; ++j) {
        const uint32_t mj = lm[j];
        const double wj = lw[j];
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (((xl | ((uint32_t)r << 8)) & mj) == mj) acc[r] = __dadd_rn(acc[r], wj);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) __stcs(out + i0 + tid + 256u * r, acc[r]);
  }
}

// compact index: idx = T - vmin when T is an integer; flags non-integral values
template <typename IDX>
__global__ void k_compact(const double* __restrict__ t, uint64_t len, double vmin, IDX* __restrict__ idx,
                          int* __restrict__ bad) {
  int local_bad = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = t[i];
    const double d = v - vmin;
    if (v != rint(v)) local_bad = 1;
    idx[i] = (IDX)d;
  }
  if (__syncthreads_or(local_bad) && threadIdx.x == 0) atomicOr(bad, 1);
}

}  // namespace

namespace qsb {

int minmax(qsb_ctx* ctx, const double* v, uint64_t len, double* mn, double* mx);  // ops.cu

// what a precompute already knows about its table (the dyadic path: min / max from the
// kernel, flip symmetry from the terms) -- finish_table skips those passes
struct TableStats {
  bool minmax = false;
  double vmin = 0, vmax = 0;
  int sym = -1;  // -1 unknown
};

static int precompute_into(qsb_ctx* ctx, const double* weights, const int64_t* masks, uint64_t num_terms,
                           double* out, uint64_t len, IndexMap map = IndexMap{63, 63, 0, 0},
                           TableStats* stats = nullptr) {
  const uint64_t tbytes = num_terms * (sizeof(double) + sizeof(uint64_t));
  QSB_TRY(ensure_small(ctx, tbytes + 64));
  double* dw = (double*)ctx->d_small;
  uint64_t* dm = (uint64_t*)(dw + num_terms);
  // dyadic weights over whole 4096-x tiles: the exact int64 subset-sum path
  const char* nz = getenv("QSB_NO_ZETA");
  const int sh = (len >= kZN && (len & (kZN - 1)) == 0 && map.b >= (uint32_t)kZT && !(nz && atoi(nz))) ? dyadic_shift(weights, num_terms) : -1;
  if (sh >= 0) {
    // exact sums: terms with equal masks merge into one (MaxCut's x_i terms repeat once
    // per edge), zero sums drop out; ascending masks put the terms of one tile-high
    // part on consecutive lanes with distinct low parts (few same-address atomics)
    std::vector<std::pair<uint64_t, long long>> tm(num_terms);
    for (uint64_t k = 0; k < num_terms; ++k) tm[k] = {(uint64_t)masks[k], (long long)ldexp(weights[k], sh)};
    std::sort(tm.begin(), tm.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    std::vector<long long> iw;
    std::vector<uint64_t> im;
    for (uint64_t k = 0; k < num_terms;) {
      uint64_t e = k;
      long long sum = 0;
      for (; e < num_terms && tm[e].first == tm[k].first; ++e) sum += tm[e].second;
      if (sum) {
        iw.push_back(sum);
        im.push_back(tm[k].first);
      }
      k = e;
    }
    const uint64_t nt = iw.size();
    if (nt) {
      QSB_CUDA(cudaMemcpyAsync(dw, iw.data(), nt * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
      QSB_CUDA(cudaMemcpyAsync(dm, im.data(), nt * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    }
    const uint64_t ntiles = len >> kZT;
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)ctx->num_sms * 4);  // <= 64 registers: 4 CTAs per SM
    QSB_TRY(ensure_scratch(ctx, 64));
    long long* dmm = (long long*)ctx->d_scratch;
    k_minmax_init<<<1, 1, 0, ctx->stream>>>(dmm);
    k_precompute_zeta<<<(unsigned)grid, kZThreads, 0, ctx->stream>>>((const long long*)dw, dm, nt, out, ntiles,
                                                                     ldexp(1.0, -sh), map, dmm);
    QSB_CHECK_LAUNCH(ctx, "precompute (dyadic)");
    long long hmm[2];
    QSB_CUDA(cudaMemcpyAsync(hmm, dmm, sizeof(hmm), cudaMemcpyDeviceToHost, ctx->stream));
    // (the host symmetry test overlaps the kernel)
    const bool identity = map.b >= 63;
    const int sym = identity ? dyadic_symmetric(im, iw) : -1;
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));  // host term arrays / d_small reuse
    if (stats) {
      stats->minmax = true;
      stats->vmin = (double)hmm[0] * ldexp(1.0, -sh);
      stats->vmax = (double)hmm[1] * ldexp(1.0, -sh);
      stats->sym = sym;
    }
    return QSB_OK;
  }
  if (num_terms) {
    // d_small may still be read by queued kernels -> synchronous, stream-ordered copies
    QSB_CUDA(cudaMemcpyAsync(dw, weights, num_terms * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    QSB_CUDA(cudaMemcpyAsync(dm, masks, num_terms * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  }
  if (len >= kZN && (len & (kZN - 1)) == 0 && map.b >= (uint32_t)kZT && !(nz && atoi(nz) > 1)) {
    // tiles of 4096 x with their terms compacted in order (QSB_NO_ZETA=2: the per-x kernel)
    const uint64_t ntiles = len >> kZT;
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)ctx->num_sms * 4);
    k_precompute_tiled<<<(unsigned)grid, kZThreads, 0, ctx->stream>>>(dw, dm, num_terms, out, ntiles, map);
    QSB_CHECK_LAUNCH(ctx, "precompute (tiled)");
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    return QSB_OK;
  }
  const uint64_t threads_needed = (len + kPreX - 1) / kPreX;
  const uint64_t blocks = (threads_needed + kPreThreads - 1) / kPreThreads;
  k_precompute<<<(unsigned)blocks, kPreThreads, 0, ctx->stream>>>(dw, dm, num_terms, out, len, map);
  QSB_CHECK_LAUNCH(ctx, "precompute");
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));  // host term arrays / d_small reuse
  return QSB_OK;
}

// flip symmetry check: bad = 1 unless v[x] == v[len-1-x] for every x
__global__ void k_symcheck(const double* __restrict__ v, uint64_t len, int* bad) {
  const uint64_t half = len >> 1;
  bool ok = true;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < half; x += (uint64_t)gridDim.x * blockDim.x)
    ok = ok && (v[x] == v[len - 1 - x]);
  if (!__syncthreads_and(ok) && threadIdx.x == 0) atomicOr(bad, 1);
}

static int finish_table(qsb_ctx* ctx, qsb_table* t, const TableStats* known = nullptr) {
  const char* nk = getenv("QSB_NO_TABLE_STATS");  // A/B + tests: recompute on the device
  if (nk && atoi(nk)) known = nullptr;
  if (known && known->minmax) {
    t->vmin = known->vmin;
    t->vmax = known->vmax;
  } else {
    QSB_TRY(minmax(ctx, t->values, t->len, &t->vmin, &t->vmax));
  }
  t->sym = 0;
  if (known && known->sym >= 0) {
    t->sym = t->len >= 2 ? known->sym : 0;
  } else if (t->len >= 2) {
    QSB_TRY(ensure_scratch(ctx, 64));
    int* bad = (int*)ctx->d_scratch;
    QSB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    k_symcheck<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(t->values, t->len, bad);
    QSB_CHECK_LAUNCH(ctx, "symmetry check");
    int hbad = 1;
    QSB_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    t->sym = hbad ? 0 : 1;
  }
  t->kind = 0;
  t->nvals = 0;
  const double range = t->vmax - t->vmin;
  const bool integral_ends = t->vmin == rint(t->vmin) && t->vmax == rint(t->vmax) && fabs(t->vmin) < 1e15 &&
                             fabs(t->vmax) < 1e15;
  if (integral_ends && range < 65536.0) {
    const int kind = range < 256.0 ? 1 : 2;
    const size_t esz = kind == 1 ? 1 : 2;
    void* idx = nullptr;
    cudaError_t e = cudaMalloc(&idx, t->len * esz);
    if (e == cudaErrorMemoryAllocation) {  // cached large blocks may be in the way
      cudaGetLastError();
      big_release(ctx->device);
      e = cudaMalloc(&idx, t->len * esz);
    }
    if (e != cudaSuccess) {  // compact table is an optimisation: fall back quietly
      cudaGetLastError();
      return QSB_OK;
    }
    QSB_TRY(ensure_scratch(ctx, 64));
    int* bad = (int*)ctx->d_scratch;
    QSB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    unsigned g = ctx->num_sms * 8;
    if (kind == 1)
      k_compact<uint8_t><<<g, 256, 0, ctx->stream>>>(t->values, t->len, t->vmin, (uint8_t*)idx, bad);
    else
      k_compact<uint16_t><<<g, 256, 0, ctx->stream>>>(t->values, t->len, t->vmin, (uint16_t*)idx, bad);
    QSB_CHECK_LAUNCH(ctx, "compact");
    int hbad = 0;
    QSB_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hbad) {
      cudaFree(idx);
      return QSB_OK;
    }
    t->cidx = idx;
    t->kind = kind;
    t->nvals = (int)range + 1;
    QSB_CUDA(dev_malloc((void**)&t->d_lut, (size_t)t->nvals * sizeof(double2), ctx->device));
    t->h_lutbuf.resize(2 * (size_t)t->nvals);
  }
  return QSB_OK;
}

// LUT entry k: extra * (cos(ang), sin(ang)), ang = ang_scale * (vmin + k), host libm
// (glibc — the functions Python's math module and numba's math.cos/sin call).
int upload_phase_lut(qsb_table* t, double ang_scale, double2 extra, bool exact) {
  qsb_ctx* ctx = t->ctx;
  double* h = t->h_lutbuf.data();
  for (int k = 0; k < t->nvals; ++k) {
    const double v = t->vmin + (double)k;
    const double ang = ang_scale * v;
    double c = cos(ang), s = sin(ang);
    if (!exact) {
      const double c2 = c * extra.x - s * extra.y;
      const double s2 = c * extra.y + s * extra.x;
      c = c2;
      s = s2;
    }
    h[2 * k] = c;
    h[2 * k + 1] = s;
  }
  // the previous LUT may still be read by a queued sweep: order on the stream,
  // and wait so the host staging buffer can be rewritten safely next time
  QSB_CUDA(cudaMemcpyAsync(t->d_lut, h, (size_t)t->nvals * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

int launch_phase_lut(qsb_ctx* ctx, qsb_table* t, double2* amps);  // ops.cu

static int wrap_table(qsb_ctx* ctx, int n, double* values, double* min_out, double* max_out, qsb_table** out,
                      const TableStats* known) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !values || !out) return invalid("qsb_table_wrap: null argument");
  if (n < 1 || n > 62) return invalid("qsb_table_wrap: n=%d out of range", n);
  qsb_table* t = new qsb_table();
  t->ctx = ctx;
  t->n = n;
  t->len = 1ull << n;
  t->values = values;
  int rc = finish_table(ctx, t, known);
  if (rc != QSB_OK) {
    qsb_table_destroy(t);
    return rc;
  }
  if (min_out) *min_out = t->vmin;
  if (max_out) *max_out = t->vmax;
  *out = t;
  return QSB_OK;
}


}  // namespace qsb

extern "C" {

int qsb_precompute_table(qsb_ctx* ctx, const double* weights, const int64_t* masks, uint64_t num_terms,
                         double* out, uint64_t len) {
  if (!ctx || !out || (num_terms && (!weights || !masks))) return invalid("qsb_precompute_table: null argument");
  if (!len) return QSB_OK;
  return precompute_into(ctx, weights, masks, num_terms, out, len);
}

int qsb_table_create(qsb_ctx* ctx, int n, const double* weights, const int64_t* masks, uint64_t num_terms,
                     double* values, double* min_out, double* max_out, qsb_table** out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !values || !out) return invalid("qsb_table_create: null argument");
  if (n < 1 || n > 62) return invalid("qsb_table_create: n=%d out of range", n);
  const uint64_t len = 1ull << n;
  for (uint64_t k = 0; k < num_terms; ++k)
    if (masks[k] < 0 || (uint64_t)masks[k] >= len) return invalid("term mask %lld out of range for n=%d", (long long)masks[k], n);
  TableStats st;
  QSB_TRY(precompute_into(ctx, weights, masks, num_terms, values, len, IndexMap{63, 63, 0, 0}, &st));
  return wrap_table(ctx, n, values, min_out, max_out, out, &st);
}

// Shard of a 2^n_global table: local index i of `rank` under the layout map
// x = (i & (2^b-1)) | (rank << s1) | ((i >> b) << s2) (see dist.py for the layouts).
int qsb_table_create_mapped(qsb_ctx* ctx, int n_global, int n_local, const double* weights, const int64_t* masks,
                            uint64_t num_terms, int b, int s1, int s2, uint64_t rank, double* values, double* min_out,
                            double* max_out, qsb_table** out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !values || !out) return invalid("qsb_table_create_mapped: null argument");
  if (n_local < 1 || n_local > n_global || n_global > 62) return invalid("bad shard geometry %d/%d", n_local, n_global);
  const uint64_t glen = 1ull << n_global;
  for (uint64_t k = 0; k < num_terms; ++k)
    if (masks[k] < 0 || (uint64_t)masks[k] >= glen)
      return invalid("term mask %lld out of range for n=%d", (long long)masks[k], n_global);
  if (b < 2 || b > n_local) return invalid("index map needs 2 <= b <= n_local (b=%d)", b);
  IndexMap map{(uint32_t)b, (uint32_t)s1, (uint32_t)s2, rank};
  TableStats st;
  QSB_TRY(precompute_into(ctx, weights, masks, num_terms, values, 1ull << n_local, map, &st));
  return wrap_table(ctx, n_local, values, min_out, max_out, out, &st);
}

int qsb_table_wrap(qsb_ctx* ctx, int n, double* values, double* min_out, double* max_out, qsb_table** out) {
  return wrap_table(ctx, n, values, min_out, max_out, out, nullptr);
}

// Does not touch t->ctx (it may already be destroyed); cudaFree synchronises.
int qsb_table_destroy(qsb_table* t) {
  if (!t) return QSB_OK;
  if (t->cidx) cudaFree(t->cidx);
  if (t->d_lut) cudaFree(t->d_lut);
  if (t->d_flut) cudaFree(t->d_flut);
  delete t;
  return QSB_OK;
}

int qsb_table_kind(qsb_table* t, int* kind, int* num_values) {
  if (!t) return invalid("null table");
  if (kind) *kind = t->kind;
  if (num_values) *num_values = t->nvals;
  return QSB_OK;
}

// Phase multiply through a table object: exact LUT path when compact
// (bit-identical to numba's glibc cos/sin), device sincos otherwise.
int qsb_table_phase(qsb_ctx* ctx, qsb_table* t, double* amps, double gamma) {
  if (!ctx || !t || !amps) return invalid("qsb_table_phase: null argument");
  if (t->kind == 0) {
    extern int qsb_phase_by_table(qsb_ctx*, double*, const double*, uint64_t, double);
    return qsb_phase_by_table(ctx, amps, t->values, t->len, gamma);
  }
  QSB_TRY(upload_phase_lut(t, -gamma, make_double2(1.0, 0.0), true));
  return launch_phase_lut(ctx, t, (double2*)amps);
}

// Host-only helper (no device needed): the LUT the library would build, for tests.
int qsb_phase_lut_host(double gamma, double vmin, int nvals, double* out) {
  if (!out || nvals < 0) return invalid("qsb_phase_lut_host: bad argument");
  for (int k = 0; k < nvals; ++k) {
    const double ang = (-gamma) * (vmin + (double)k);
    out[2 * k] = cos(ang);
    out[2 * k + 1] = sin(ang);
  }
  return QSB_OK;
}

}  // extern "C"
