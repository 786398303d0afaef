// Shot sampling (backend.sample_indices, backend.py:261-299; sampling.draw,
// sampling.py:23-30).
//
// The reference builds every pairwise level of the probability tree
// (leaves |psi_i|^2, level l+1 = src[2i] + src[2i+1]) and descends it once per
// shot with a splitmix64 uniform scaled by the root.  The GPU builds the same
// levels with the same association (11 levels per launch: 3 in registers, 5 by
// warp shuffle, 3 through shared memory) but stores only levels k0..n (k0 = 5:
// 1/16 of the tree, 512 MB at n=30); one thread per shot descends the stored
// levels, then rebuilds its 32-leaf subtree from the amplitudes (the same adds in
// the same order) for the last k0 steps.  Every floating-point operation matches
// the reference, so given the same state the drawn indices are bit-identical.
#include <math.h>

#include "common.cuh"

using namespace qsb;
using namespace qsbd;

namespace {

constexpr int kBT = 256;        // threads per build block
constexpr int kBPer = 8;        // inputs per thread
constexpr int kBIn = kBT * kBPer;  // 2048 inputs per block -> 11 levels

constexpr int kK0 = 5;  // lowest stored level (below: rebuilt per shot from 2^k0 leaves)

struct Levels {
  double* base;
  uint64_t N;
  int n;
  int k0;  // min(kK0, n)
  // level l >= k0 starts at sum_{k=k0}^{l-1} N >> k = (N >> (k0-1)) - (N >> (l-1))
  __host__ __device__ uint64_t off(int l) const { return (N >> (k0 - 1)) - (N >> (l - 1)); }
  __host__ __device__ bool stored(int l) const { return l >= k0 && l <= n; }
  // entries of levels k0..n
  __host__ __device__ uint64_t count() const { return (N >> (k0 - 1)) - (N >> n); }
};

// Build levels l0+1 .. l0+11 (those <= n) from level l0 (l0 == 0: from amplitudes).
__global__ void __launch_bounds__(kBT) k_build(const double2* __restrict__ amps, Levels L, int l0) {
  __shared__ double sh[kBT / 32];
  const uint64_t M = L.N >> l0;  // number of inputs at level l0
  const uint64_t i0 = (uint64_t)blockIdx.x * kBIn + (uint64_t)threadIdx.x * kBPer;
  double r[kBPer];
  const double* src = l0 > 0 ? L.base + L.off(l0) : nullptr;
#pragma unroll
  for (int e = 0; e < kBPer; ++e) {
    const uint64_t i = i0 + e;
    if (i < M) r[e] = l0 == 0 ? norm2_exact(amps[i]) : src[i];
    else r[e] = 0.0;
  }
  // register levels 1..3
  int lvl = l0;
#pragma unroll
  for (int w = kBPer / 2, k = 1; w >= 1; w >>= 1, ++k) {
#pragma unroll
    for (int e = 0; e < w; ++e) r[e] = __dadd_rn(r[2 * e], r[2 * e + 1]);
    const int l = l0 + k;
    if (L.stored(l)) {
      const uint64_t cnt = L.N >> l;
      double* dst = L.base + L.off(l);
      const uint64_t j0 = (i0 >> k);
#pragma unroll
      for (int e = 0; e < w; ++e)
        if (j0 + e < cnt) dst[j0 + e] = r[e];
    }
    lvl = l;
  }
  double v = r[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // shuffle levels: lane groups of 2,4,...,32
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1 << k));
    const int l = lvl + 1 + k;
    if (L.stored(l) && (lane & ((2 << k) - 1)) == 0) {
      const uint64_t cnt = L.N >> l;
      const uint64_t j = (i0 >> 3) >> (k + 1);
      if (j < cnt) L.base[L.off(l) + j] = v;
    }
  }
  lvl += 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double w8[kBT / 32];
#pragma unroll
    for (int e = 0; e < kBT / 32; ++e) w8[e] = sh[e];
    int k = 0;
#pragma unroll
    for (int w = kBT / 64; w >= 1; w >>= 1, ++k) {
#pragma unroll
      for (int e = 0; e < w; ++e) w8[e] = __dadd_rn(w8[2 * e], w8[2 * e + 1]);
      const int l = lvl + 1 + k;
      if (L.stored(l)) {
        const uint64_t cnt = L.N >> l;
        const uint64_t j0 = (uint64_t)blockIdx.x * w;
        for (int e = 0; e < w; ++e)
          if (j0 + e < cnt) L.base[L.off(l) + j0 + e] = w8[e];
      }
    }
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// the cost of a drawn index: the fp64 table, or (a sharded table whose fp64 copy was
// dropped, qsb_table_detach_values) the compact index: T = vmin + idx, exact for the
// integral tables that have one
struct CostView {
  const double* values;
  const void* cidx;
  int kind;
  double vmin;
  __device__ double at(uint64_t i) const {
    if (values) return values[i];
    return vmin + (double)(kind == 1 ? ((const uint8_t*)cidx)[i] : ((const uint16_t*)cidx)[i]);
  }
};

// u_in == nullptr: u_s = U(seed, s) * root (the reference's draw); else u_s = u_in[s]
// (a shard's residuals after the caller descended the levels above it).
// half != 0 (a flip-symmetric state, Z2 reduction): amps and the stored levels hold
// only the lower half x < N/2 of the full n-qubit tree.  Every node of the upper half
// equals its mirror: full level-l node j == node N_l - 1 - j (pairwise sums of the
// reversed leaves, and IEEE addition is commutative), so a lookup of node j reads the
// lower-half node min(j, N_l - 1 - j) and a leaf x >= N/2 reads amplitude N - 1 - x.
// L.n is the full tree's height; the root level is the caller's (h + h).
__global__ void k_descend(const double2* __restrict__ amps, Levels L, const CostView table, uint64_t shots,
                          uint64_t seed, double root, const double* __restrict__ u_in, int64_t* __restrict__ idx_out,
                          double* __restrict__ cost_out, int half) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < shots; s += (uint64_t)gridDim.x * blockDim.x) {
    double u;
    if (u_in) {
      u = u_in[s];
    } else {
      // rng.uniform_block(seed, 0, shots)[s] * total  (rng.py:40-47, backend.py:291)
      const uint64_t z = mix64(seed + (s + 1) * 0x9E3779B97F4A7C15ull);
      u = __dmul_rn(__dmul_rn((double)(z >> 11), 0x1.0p-53), root);
    }
    uint64_t idx = 0;  // node at level l+1
    for (int l = L.n - 1; l >= L.k0; --l) {
      uint64_t j = 2 * idx;
      if (half) {
        const uint64_t nl = (L.N << 1) >> l;  // full-tree nodes at level l
        if (j >= nl >> 1) j = nl - 1 - j;
      }
      const double left = L.base[L.off(l) + j];
      const bool right = u >= left;
      if (right) u = __dadd_rn(u, -left);
      idx = 2 * idx + (right ? 1 : 0);
    }
    // idx is a node of level k0: rebuild its subtree (levels 0..k0-1) from the
    // 2^k0 amplitudes below it, exactly as the reference's levels were formed
    double t[2 << kK0];  // t[0..2^k0) leaves, then level 1, level 2, ... packed
    const int k0 = L.k0;
    const uint64_t leaf0 = idx << k0;
#pragma unroll
    for (int e = 0; e < (1 << kK0); ++e)
      if (e < (1 << k0)) {
        uint64_t x = leaf0 + e;
        if (half && x >= L.N) x = 2 * L.N - 1 - x;
        t[e] = norm2_exact(amps[x]);
      }
    int lo[kK0 + 1];
    lo[0] = 0;
#pragma unroll
    for (int l = 1; l <= kK0; ++l) {
      lo[l] = lo[l - 1] + (1 << (kK0 - l + 1));
      if (l < k0) {
#pragma unroll
        for (int e = 0; e < (1 << (kK0 - l)); ++e)
          if (e < (1 << (k0 - l))) t[lo[l] + e] = __dadd_rn(t[lo[l - 1] + 2 * e], t[lo[l - 1] + 2 * e + 1]);
      }
    }
    uint64_t loc = 0;  // node within the subtree at level l+1
#pragma unroll
    for (int l = kK0 - 1; l >= 0; --l) {
      if (l < k0) {
        const double left = t[lo[l] + 2 * loc];
        const bool right = u >= left;
        if (right && l > 0) u = __dadd_rn(u, -left);
        loc = 2 * loc + (right ? 1 : 0);
      }
    }
    idx = leaf0 + loc;
    idx_out[s] = (int64_t)idx;
    if (cost_out) cost_out[s] = table.at(idx);
  }
}

// Build the stored levels of the n-qubit state's probability tree into the context's
// sampler scratch; *root = its root (the total probability).
int build_tree(qsb_ctx* ctx, const double2* a, int n, Levels* Lout, double* root) {
  const uint64_t N = 1ull << n;
  const int k0 = n < kK0 ? n : kK0;
  Levels L{nullptr, N, n, k0};
  QSB_TRY(ensure_sample_scratch(ctx, L.count() * sizeof(double)));
  L.base = (double*)ctx->d_sample;
  for (int l0 = 0; l0 < n; l0 += 11) {
    const uint64_t M = N >> l0;
    const uint64_t blocks = (M + kBIn - 1) / kBIn;
    k_build<<<(unsigned)blocks, kBT, 0, ctx->stream>>>(a, L, l0);
    QSB_CHECK_LAUNCH(ctx, "sample tree build");
  }
  QSB_CUDA(cudaMemcpyAsync(ctx->h_small, L.base + L.off(n), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->d2h_bytes += sizeof(double);
  *root = ctx->h_small[0];
  *Lout = L;
  return QSB_OK;
}

// Descend `shots` shots on the tree in L (uniforms from the seed, or u_host); indices
// and costs copied to the host arrays.
int descend(qsb_ctx* ctx, qsb_table* t, const double2* a, const Levels& L, uint64_t shots, uint64_t seed, double root,
            const double* u_host, int64_t* idx_out, double* cost_out, int half = 0) {
  QSB_TRY(ensure_shot_scratch(ctx, shots * (sizeof(int64_t) + sizeof(double) + (u_host ? sizeof(double) : 0))));
  int64_t* d_idx = (int64_t*)ctx->d_shots;
  double* d_cost = (double*)(d_idx + shots);
  double* d_u = u_host ? d_cost + shots : nullptr;
  if (u_host) {
    QSB_CUDA(cudaMemcpyAsync(d_u, u_host, shots * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += shots * sizeof(double);
  }
  uint64_t blocks = (shots + 255) / 256;
  if (blocks > (uint64_t)ctx->num_sms * 64) blocks = (uint64_t)ctx->num_sms * 64;
  const CostView cv{t ? t->values : nullptr, t ? t->cidx : nullptr, t ? t->kind : 0, t ? t->vmin : 0.0};
  if (t && !t->values && !t->cidx) return invalid("sampling: the table has neither fp64 values nor a compact index");
  k_descend<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, L, cv, shots, seed, root, d_u, d_idx, t ? d_cost : nullptr,
                                                       half);
  QSB_CHECK_LAUNCH(ctx, "sample descent");
  QSB_CUDA(cudaMemcpyAsync(idx_out, d_idx, shots * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  if (t) QSB_CUDA(cudaMemcpyAsync(cost_out, d_cost, shots * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->d2h_bytes += shots * (sizeof(int64_t) + (t ? sizeof(double) : 0));
  return QSB_OK;
}

}  // namespace

extern "C" {

int qsb_sample(qsb_ctx* ctx, qsb_table* t, const double* amps, int n, uint64_t shots, uint64_t seed,
               int64_t* idx_out, double* cost_out, double* total_out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !amps || !idx_out) return invalid("qsb_sample: null argument");
  if (shots < 1) return invalid("shots must be >= 1, got %llu", (unsigned long long)shots);
  if (n < 1 || n > 62) return invalid("qsb_sample: n=%d out of range", n);
  if (t && n != t->n) return invalid("qsb_sample: state has n=%d, table n=%d", n, t->n);
  if (t && !cost_out) return invalid("qsb_sample: table given without a cost output");
  const double2* a = (const double2*)amps;
  Levels L;
  double root;
  ctx->tree_n = -1;  // the scratch no longer holds a qsb_sample_tree tree
  QSB_TRY(build_tree(ctx, a, n, &L, &root));
  if (total_out) *total_out = root;
  if (!(fabs(root - 1.0) <= 1e-9)) return invalid("state is not normalized: sum of probabilities = %.17g", root);
  return descend(ctx, t, a, L, shots, seed, root, nullptr, idx_out, cost_out);
}

int qsb_sample_sym(qsb_ctx* ctx, qsb_table* t, const double* half_amps, int n, uint64_t shots, uint64_t seed,
                   int64_t* idx_out, double* cost_out, double* total_out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !half_amps || !idx_out) return invalid("qsb_sample_sym: null argument");
  if (shots < 1) return invalid("shots must be >= 1, got %llu", (unsigned long long)shots);
  if (n < 2 || n > 62) return invalid("qsb_sample_sym: n=%d out of range", n);
  if (t && n != t->n) return invalid("qsb_sample_sym: state has n=%d, table n=%d", n, t->n);
  if (t && !cost_out) return invalid("qsb_sample_sym: table given without a cost output");
  const double2* a = (const double2*)half_amps;
  Levels L;
  double h;
  ctx->tree_n = -1;
  QSB_TRY(build_tree(ctx, a, n - 1, &L, &h));  // levels 0..n-1 of the lower half
  const double root = h + h;                   // full level n: lower root + its mirror
  if (total_out) *total_out = root;
  if (!(fabs(root - 1.0) <= 1e-9)) return invalid("state is not normalized: sum of probabilities = %.17g", root);
  Levels F = L;
  F.n = n;  // the full tree's height (node lookups fold into the stored half)
  return descend(ctx, t, a, F, shots, seed, root, nullptr, idx_out, cost_out, 1);
}

int qsb_sample_tree(qsb_ctx* ctx, const double* amps, int n_local, double* root_out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !amps || !root_out) return invalid("qsb_sample_tree: null argument");
  if (n_local < 1 || n_local > 62) return invalid("qsb_sample_tree: n=%d out of range", n_local);
  Levels L;
  QSB_TRY(build_tree(ctx, (const double2*)amps, n_local, &L, root_out));
  ctx->tree_n = n_local;
  ctx->tree_amps = amps;
  return QSB_OK;
}

int qsb_sample_descend(qsb_ctx* ctx, qsb_table* t, const double* amps, int n_local, uint64_t count, const double* u,
                       int64_t* idx_out, double* cost_out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !amps || (count && (!u || !idx_out))) return invalid("qsb_sample_descend: null argument");
  if (ctx->tree_n != n_local || ctx->tree_amps != amps)
    return invalid("qsb_sample_descend: no tree for this state (call qsb_sample_tree first)");
  if (t && n_local != t->n) return invalid("qsb_sample_descend: shard has n=%d, table n=%d", n_local, t->n);
  if (t && count && !cost_out) return invalid("qsb_sample_descend: table given without a cost output");
  if (count == 0) return QSB_OK;
  const uint64_t N = 1ull << n_local;
  const int k0 = n_local < kK0 ? n_local : kK0;
  Levels L{(double*)ctx->d_sample, N, n_local, k0};
  return descend(ctx, t, (const double2*)amps, L, count, 0, 0.0, u, idx_out, cost_out);
}

}  // extern "C"
