// Shot sampling (backend.sample_indices, backend.py:261-299; sampling.draw,
// sampling.py:23-30).
//
// The reference builds every pairwise level of the probability tree
// (leaves |psi_i|^2, level l+1 = src[2i] + src[2i+1]) and descends it once per
// shot with a splitmix64 uniform scaled by the root.  The GPU builds the same
// levels 1..n with the same association (11 levels per launch: 3 in registers,
// 5 by warp shuffle, 3 through shared memory), never stores the leaves (they are
// recomputed from two amplitudes at the bottom of the descent), then runs one
// thread per shot.  Every floating-point operation matches the reference, so
// given the same state the drawn indices are bit-identical.
#include <math.h>

#include "common.cuh"

using namespace qsb;
using namespace qsbd;

namespace {

constexpr int kBT = 256;        // threads per build block
constexpr int kBPer = 8;        // inputs per thread
constexpr int kBIn = kBT * kBPer;  // 2048 inputs per block -> 11 levels

struct Levels {
  double* base;
  uint64_t N;
  int n;
  // level l >= 1 starts at sum_{k=1}^{l-1} N >> k = N - (N >> (l-1)); the root is at N - 2
  __host__ __device__ uint64_t off(int l) const { return N - (N >> (l - 1)); }
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
    if (l <= L.n) {
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
    if (l <= L.n && (lane & ((2 << k) - 1)) == 0) {
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
      if (l <= L.n) {
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

__global__ void k_descend(const double2* __restrict__ amps, Levels L, const double* __restrict__ table, uint64_t shots,
                          uint64_t seed, double root, int64_t* __restrict__ idx_out, double* __restrict__ cost_out) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < shots; s += (uint64_t)gridDim.x * blockDim.x) {
    // rng.uniform_block(seed, 0, shots)[s] * total  (rng.py:40-47, backend.py:291)
    const uint64_t z = mix64(seed + (s + 1) * 0x9E3779B97F4A7C15ull);
    double u = __dmul_rn(__dmul_rn((double)(z >> 11), 0x1.0p-53), root);
    uint64_t idx = 0;
    for (int l = L.n - 1; l >= 1; --l) {
      const double left = L.base[L.off(l) + 2 * idx];
      const bool right = u >= left;
      if (right) u = __dadd_rn(u, -left);
      idx = 2 * idx + (right ? 1 : 0);
    }
    {
      const double left = norm2_exact(amps[2 * idx]);
      const bool right = u >= left;
      idx = 2 * idx + (right ? 1 : 0);
    }
    idx_out[s] = (int64_t)idx;
    if (table) cost_out[s] = table[idx];
  }
}

}  // namespace

extern "C" {

int qsb_sample(qsb_ctx* ctx, qsb_table* t, const double* amps, int n, uint64_t shots, uint64_t seed,
               int64_t* idx_out, double* cost_out, double* total_out) {
  if (!ctx || !amps || !idx_out) return invalid("qsb_sample: null argument");
  if (shots < 1) return invalid("shots must be >= 1, got %llu", (unsigned long long)shots);
  if (n < 1 || n > 62) return invalid("qsb_sample: n=%d out of range", n);
  if (t && n != t->n) return invalid("qsb_sample: state has n=%d, table n=%d", n, t->n);
  if (t && !cost_out) return invalid("qsb_sample: table given without a cost output");
  const uint64_t N = 1ull << n;
  const double2* a = (const double2*)amps;
  double root;
  double* levels = nullptr;
  int64_t* d_idx = nullptr;
  double* d_cost = nullptr;
  const uint64_t lv_count = N > 1 ? N - 1 : 1;
  QSB_CUDA(cudaMallocAsync((void**)&levels, lv_count * sizeof(double), ctx->stream));
  Levels L{levels, N, n};
  int rc = QSB_OK;
  for (int l0 = 0; l0 < n; l0 += 11) {
    const uint64_t M = N >> l0;
    const uint64_t blocks = (M + kBIn - 1) / kBIn;
    k_build<<<(unsigned)blocks, kBT, 0, ctx->stream>>>(a, L, l0);
    ctx->launches++;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) rc = cuda_fail(e, "sample tree build");
  if (rc == QSB_OK) {
    e = cudaMemcpyAsync(ctx->h_small, levels + L.off(n), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "sample root");
  }
  if (rc == QSB_OK) {
    root = ctx->h_small[0];
    if (total_out) *total_out = root;
    if (!(fabs(root - 1.0) <= 1e-9)) rc = invalid("state is not normalized: sum of probabilities = %.17g", root);
  }
  if (rc == QSB_OK) {
    e = cudaMallocAsync((void**)&d_idx, shots * sizeof(int64_t), ctx->stream);
    if (e == cudaSuccess && t) e = cudaMallocAsync((void**)&d_cost, shots * sizeof(double), ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "sample output allocation");
  }
  if (rc == QSB_OK) {
    uint64_t blocks = (shots + 255) / 256;
    if (blocks > (uint64_t)ctx->num_sms * 64) blocks = (uint64_t)ctx->num_sms * 64;
    k_descend<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a, L, t ? t->values : nullptr, shots, seed, root, d_idx, d_cost);
    ctx->launches++;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(idx_out, d_idx, shots * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && t) e = cudaMemcpyAsync(cost_out, d_cost, shots * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "sample descent");
    ctx->d2h_bytes += shots * (sizeof(int64_t) + (t ? sizeof(double) : 0)) + sizeof(double);
  }
  if (d_idx) cudaFreeAsync(d_idx, ctx->stream);
  if (d_cost) cudaFreeAsync(d_cost, ctx->stream);
  cudaFreeAsync(levels, ctx->stream);
  return rc;
}

}  // extern "C"
