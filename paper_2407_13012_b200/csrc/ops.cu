// The 14-function kernel set (mirror of qaoasim/kernels/numba_impl.py) on device
// buffers.  Arithmetic is FMA-free and associations follow the reference, so the
// results are bit-identical to the numba set on identical inputs; the only
// exception is phase_by_table on a non-integral table (device sincos, <= 2 ulp).
#include <math.h>

#include "common.cuh"

using namespace qsb;
using namespace qsbd;

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t work, int per_thread = 1) {
  uint64_t blocks = (work + (uint64_t)kThreads * per_thread - 1) / ((uint64_t)kThreads * per_thread);
  if (blocks < 1) blocks = 1;
  if (blocks > (1u << 30)) blocks = (1u << 30);
  return (unsigned)blocks;
}

// grid-stride index helper
#define GRID_LOOP(i, n) \
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_fill_plus(double2* amps, uint64_t len, double v) {
  GRID_LOOP(i, len) amps[i] = make_double2(v, 0.0);
}

// numba: ang = -gamma * table[i]; amps[i] *= complex(cos(ang), sin(ang))
__global__ void k_phase_sincos(double2* amps, const double* table, uint64_t len, double neg_gamma) {
  GRID_LOOP(i, len) {
    double ang = __dmul_rn(neg_gamma, table[i]);
    double s, c;
    sincos(ang, &s, &c);
    amps[i] = cmul_exact(amps[i], make_double2(c, s));
  }
}

template <typename IDX>
__global__ void k_phase_lut(double2* amps, const IDX* cidx, uint64_t len, const double2* lut) {
  GRID_LOOP(i, len) amps[i] = cmul_exact(amps[i], __ldg(&lut[cidx[i]]));
}

__global__ void k_diag_scale(double2* amps, const double* table, uint64_t len) {
  GRID_LOOP(i, len) {
    double2 a = amps[i];
    double t = table[i];
    amps[i] = make_double2(__dmul_rn(a.x, t), __dmul_rn(a.y, t));
  }
}

// numba_impl.rx_qubit: pairs (i0, i0|2^j); new0 = c*t + (-is)*u, new1 = (-is)*t + c*u
__global__ void k_rx_qubit(double2* amps, uint64_t half, int j, double c, double s) {
  const uint64_t low = (1ull << j) - 1ull;
  const uint64_t bit = 1ull << j;
  GRID_LOOP(k, half) {
    uint64_t i0 = ((k & ~low) << 1) | (k & low);
    uint64_t i1 = i0 | bit;
    double2 t = amps[i0], u = amps[i1];
    amps[i0] = make_double2(__dadd_rn(__dmul_rn(c, t.x), __dmul_rn(s, u.y)),
                            __dadd_rn(__dmul_rn(c, t.y), -__dmul_rn(s, u.x)));
    amps[i1] = make_double2(__dadd_rn(__dmul_rn(s, t.y), __dmul_rn(c, u.x)),
                            __dadd_rn(__dmul_rn(c, u.y), -__dmul_rn(s, t.x)));
  }
}

__global__ void k_weighted_probs(const double2* amps, const double* table, double* out, uint64_t len) {
  GRID_LOOP(i, len) out[i] = __dmul_rn(table[i], norm2_exact(amps[i]));
}

__global__ void k_probs(const double2* amps, double* out, uint64_t len) {
  GRID_LOOP(i, len) out[i] = norm2_exact(amps[i]);
}

__global__ void k_pairwise_level(const double* src, double* dst, uint64_t dst_len) {
  GRID_LOOP(i, dst_len) dst[i] = __dadd_rn(src[2 * i], src[2 * i + 1]);
}

// ---------------------------------------------------------------- exact trees
// One CTA folds a 2048-element aligned block with the neighbour-pair tree
// (8 per thread in registers, 5 shuffle levels, 3 shared-memory levels).
// Because blocks are aligned powers of two, the per-block sums are exactly the
// level-11 nodes of the reference's full tree; folding the partials with the
// same kernel (zero padding at the tail) completes that tree
// (numba_impl.py:89-126, numpy_impl.py:78-84).
constexpr int kTreeBlock = 2048;
constexpr int kTreePer = 8;

template <int NC>
struct Vals { double v[NC]; };

struct LoadPlain {
  const double* p;
  __device__ Vals<1> operator()(uint64_t i) const { return {{p[i]}}; }
};
struct LoadPair {  // two planar component arrays
  const double* p0; const double* p1;
  __device__ Vals<2> operator()(uint64_t i) const { return {{p0[i], p1[i]}}; }
};
struct LoadWeighted {
  const double2* a; const double* t;
  __device__ Vals<1> operator()(uint64_t i) const { return {{__dmul_rn(t[i], norm2_exact(a[i]))}}; }
};
struct LoadInner {
  const double2* a; const double2* b;
  __device__ Vals<2> operator()(uint64_t i) const {
    double2 x = a[i], y = b[i];
    return {{re_conj_mul_exact(x, y), im_conj_mul_exact(x, y)}};
  }
};
struct LoadDiagInner {
  const double2* a; const double* t; const double2* b;
  __device__ Vals<2> operator()(uint64_t i) const {
    double2 x = a[i], y = b[i];
    double w = t[i];
    return {{__dmul_rn(re_conj_mul_exact(x, y), w), __dmul_rn(im_conj_mul_exact(x, y), w)}};
  }
};
struct LoadXsum {
  const double2* a; const double2* b; uint64_t bit;
  __device__ Vals<2> operator()(uint64_t i) const {
    double2 x = a[i], y = b[i ^ bit];
    return {{re_conj_mul_exact(x, y), im_conj_mul_exact(x, y)}};
  }
};

// out layout: out[c * out_stride + block]
template <int NC, class F>
__global__ void __launch_bounds__(kTreeBlock / kTreePer)
k_tree_blocks(F f, uint64_t len, double* out, uint64_t out_stride) {
  __shared__ double sh[NC][kTreeBlock / kTreePer / 32];
  const uint64_t block = blockIdx.x;
  const uint64_t base = block * kTreeBlock + (uint64_t)threadIdx.x * kTreePer;
  double r[NC][kTreePer];
#pragma unroll
  for (int e = 0; e < kTreePer; ++e) {
    if (base + e < len) {
      Vals<NC> v = f(base + e);
#pragma unroll
      for (int c = 0; c < NC; ++c) r[c][e] = v.v[c];
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) r[c][e] = 0.0;
    }
  }
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
#pragma unroll
    for (int w = kTreePer / 2; w >= 1; w >>= 1)
#pragma unroll
      for (int e = 0; e < w; ++e) r[c][e] = __dadd_rn(r[c][2 * e], r[c][2 * e + 1]);
    acc[c] = r[c][0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) acc[c] = __dadd_rn(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) sh[c][warp] = acc[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    constexpr int NW = kTreeBlock / kTreePer / 32;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double w8[NW];
#pragma unroll
      for (int e = 0; e < NW; ++e) w8[e] = sh[c][e];
#pragma unroll
      for (int w = NW / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int e = 0; e < w; ++e) w8[e] = __dadd_rn(w8[2 * e], w8[2 * e + 1]);
      out[c * out_stride + block] = w8[0];
    }
  }
}

// min/max (order-free, exact)
__global__ void k_minmax_blocks(const double* v, uint64_t len, double* out_min, double* out_max) {
  __shared__ double smin[32], smax[32];
  double mn = INFINITY, mx = -INFINITY;
  GRID_LOOP(i, len) {
    double x = v[i];
    mn = fmin(mn, x);
    mx = fmax(mx, x);
  }
  for (int o = 16; o >= 1; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { smin[warp] = mn; smax[warp] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mn = fmin(mn, smin[w]); mx = fmax(mx, smax[w]); }
    out_min[blockIdx.x] = mn;
    out_max[blockIdx.x] = mx;
  }
}

}  // namespace

namespace qsb {

// Full exact tree over `len` elements produced by f; result(s) copied to host.
template <int NC, class F>
int tree_reduce(qsb_ctx* ctx, F f, uint64_t len, double* host_out) {
  if (len == 0) return invalid("tree reduction over an empty buffer");
  uint64_t nb = (len + kTreeBlock - 1) / kTreeBlock;
  // scratch: two ping-pong partial arrays of NC * nb doubles
  QSB_TRY(ensure_scratch(ctx, 2 * NC * nb * sizeof(double) + 64));
  double* a = ctx->d_scratch;
  double* b = ctx->d_scratch + NC * nb;
  k_tree_blocks<NC, F><<<(unsigned)nb, kTreeBlock / kTreePer, 0, ctx->stream>>>(f, len, a, nb);
  QSB_CHECK_LAUNCH(ctx, "tree_blocks");
  uint64_t cur = nb, stride = nb;
  while (cur > 1) {
    uint64_t nb2 = (cur + kTreeBlock - 1) / kTreeBlock;
    if constexpr (NC == 1) {
      k_tree_blocks<1, LoadPlain><<<(unsigned)nb2, kTreeBlock / kTreePer, 0, ctx->stream>>>(LoadPlain{a}, cur, b, nb2);
    } else {
      k_tree_blocks<2, LoadPair><<<(unsigned)nb2, kTreeBlock / kTreePer, 0, ctx->stream>>>(
          LoadPair{a, a + stride}, cur, b, nb2);
    }
    QSB_CHECK_LAUNCH(ctx, "tree_fold");
    double* t = a; a = b; b = t;
    cur = nb2;
    stride = nb2;
  }
  for (int c = 0; c < NC; ++c)
    QSB_CUDA(cudaMemcpyAsync(ctx->h_small + c, a + c * stride, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += NC * sizeof(double);
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int c = 0; c < NC; ++c) host_out[c] = ctx->h_small[c];
  return QSB_OK;
}

int minmax(qsb_ctx* ctx, const double* v, uint64_t len, double* mn, double* mx) {
  if (len == 0) return invalid("min/max over an empty buffer");
  unsigned nb = grid_for(len, 8);
  if (nb > (unsigned)ctx->num_sms * 8) nb = ctx->num_sms * 8;
  QSB_TRY(ensure_scratch(ctx, 2ull * nb * sizeof(double)));
  k_minmax_blocks<<<nb, kThreads, 0, ctx->stream>>>(v, len, ctx->d_scratch, ctx->d_scratch + nb);
  QSB_CHECK_LAUNCH(ctx, "minmax");
  std::vector<double> h(2 * nb);
  QSB_CUDA(cudaMemcpyAsync(h.data(), ctx->d_scratch, 2ull * nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  double a = h[0], b = h[nb];
  for (unsigned i = 1; i < nb; ++i) { a = fmin(a, h[i]); b = fmax(b, h[nb + i]); }
  *mn = a;
  *mx = b;
  return QSB_OK;
}

int launch_phase_lut(qsb_ctx* ctx, qsb_table* t, double2* amps) {
  unsigned g = grid_for(t->len, 4);
  if (t->kind == 1)
    k_phase_lut<uint8_t><<<g, kThreads, 0, ctx->stream>>>(amps, (const uint8_t*)t->cidx, t->len, t->d_lut);
  else
    k_phase_lut<uint16_t><<<g, kThreads, 0, ctx->stream>>>(amps, (const uint16_t*)t->cidx, t->len, t->d_lut);
  QSB_CHECK_LAUNCH(ctx, "phase_lut");
  return QSB_OK;
}

int launch_phase_sincos(qsb_ctx* ctx, double2* amps, const double* table, uint64_t len, double gamma) {
  k_phase_sincos<<<grid_for(len, 4), kThreads, 0, ctx->stream>>>(amps, table, len, -gamma);
  QSB_CHECK_LAUNCH(ctx, "phase_sincos");
  return QSB_OK;
}

int launch_rx_qubit(qsb_ctx* ctx, double2* amps, uint64_t len, int j, double c, double s) {
  uint64_t half = len >> 1;
  if (half == 0) return QSB_OK;
  k_rx_qubit<<<grid_for(half, 4), kThreads, 0, ctx->stream>>>(amps, half, j, c, s);
  QSB_CHECK_LAUNCH(ctx, "rx_qubit");
  return QSB_OK;
}

int launch_fill_plus(qsb_ctx* ctx, double2* amps, uint64_t len) {
  double v = 1.0 / sqrt((double)len);  // numba_impl.py:42 (host libm sqrt, correctly rounded)
  k_fill_plus<<<grid_for(len, 4), kThreads, 0, ctx->stream>>>(amps, len, v);
  QSB_CHECK_LAUNCH(ctx, "fill_plus");
  return QSB_OK;
}

int expectation_exact(qsb_ctx* ctx, const double* table, const double2* amps, uint64_t len, double* out) {
  return tree_reduce<1>(ctx, LoadWeighted{amps, table}, len, out);
}

int diag_inner_exact(qsb_ctx* ctx, const double2* a, const double* table, const double2* b, uint64_t len,
                     double* out2) {
  return tree_reduce<2>(ctx, LoadDiagInner{a, table, b}, len, out2);
}

int xsum_exact(qsb_ctx* ctx, const double2* a, const double2* b, uint64_t len, int nq, double* out2) {
  double re = 0.0, im = 0.0;  // total = 0+0j; total += complex(...) per qubit, ascending
  for (int j = 0; j < nq; ++j) {
    double r[2];
    QSB_TRY(tree_reduce<2>(ctx, LoadXsum{a, b, 1ull << j}, len, r));
    re += r[0];
    im += r[1];
  }
  out2[0] = re;
  out2[1] = im;
  return QSB_OK;
}

}  // namespace qsb

extern "C" {

int qsb_fill_plus(qsb_ctx* ctx, double* amps, uint64_t len) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !amps) return invalid("qsb_fill_plus: null argument");
  if (!len) return QSB_OK;
  return launch_fill_plus(ctx, (double2*)amps, len);
}

int qsb_phase_by_table(qsb_ctx* ctx, double* amps, const double* table, uint64_t len, double gamma) {
  if (!ctx || !amps || !table) return invalid("qsb_phase_by_table: null argument");
  if (!len) return QSB_OK;
  return launch_phase_sincos(ctx, (double2*)amps, table, len, gamma);
}

int qsb_diag_scale(qsb_ctx* ctx, double* amps, const double* table, uint64_t len) {
  if (!ctx || !amps || !table) return invalid("qsb_diag_scale: null argument");
  if (!len) return QSB_OK;
  k_diag_scale<<<grid_for(len, 4), kThreads, 0, ctx->stream>>>((double2*)amps, table, len);
  QSB_CHECK_LAUNCH(ctx, "diag_scale");
  return QSB_OK;
}

int qsb_rx_qubit(qsb_ctx* ctx, double* amps, uint64_t len, int j, double c, double s) {
  if (!ctx || !amps) return invalid("qsb_rx_qubit: null argument");
  if (j < 0 || (len >> j) < 2) return invalid("qsb_rx_qubit: qubit %d out of range for length %llu", j,
                                              (unsigned long long)len);
  return launch_rx_qubit(ctx, (double2*)amps, len, j, c, s);
}

int qsb_weighted_probs(qsb_ctx* ctx, const double* amps, const double* table, double* out, uint64_t len) {
  if (!ctx || !amps || !table || !out) return invalid("qsb_weighted_probs: null argument");
  if (!len) return QSB_OK;
  k_weighted_probs<<<grid_for(len, 4), kThreads, 0, ctx->stream>>>((const double2*)amps, table, out, len);
  QSB_CHECK_LAUNCH(ctx, "weighted_probs");
  return QSB_OK;
}

int qsb_probs(qsb_ctx* ctx, const double* amps, double* out, uint64_t len) {
  if (!ctx || !amps || !out) return invalid("qsb_probs: null argument");
  if (!len) return QSB_OK;
  k_probs<<<grid_for(len, 4), kThreads, 0, ctx->stream>>>((const double2*)amps, out, len);
  QSB_CHECK_LAUNCH(ctx, "probs");
  return QSB_OK;
}

int qsb_tree_sum(qsb_ctx* ctx, const double* vals, uint64_t len, double* out) {
  if (!ctx || !vals || !out) return invalid("qsb_tree_sum: null argument");
  return tree_reduce<1>(ctx, LoadPlain{vals}, len, out);
}

int qsb_reduce_min(qsb_ctx* ctx, const double* vals, uint64_t len, double* out) {
  if (!ctx || !vals || !out) return invalid("qsb_reduce_min: null argument");
  double mx;
  return minmax(ctx, vals, len, out, &mx);
}

int qsb_reduce_max(qsb_ctx* ctx, const double* vals, uint64_t len, double* out) {
  if (!ctx || !vals || !out) return invalid("qsb_reduce_max: null argument");
  double mn;
  return minmax(ctx, vals, len, &mn, out);
}

int qsb_inner(qsb_ctx* ctx, const double* a, const double* b, uint64_t len, double out[2]) {
  if (!ctx || !a || !b || !out) return invalid("qsb_inner: null argument");
  return tree_reduce<2>(ctx, LoadInner{(const double2*)a, (const double2*)b}, len, out);
}

int qsb_diag_inner(qsb_ctx* ctx, const double* a, const double* table, const double* b, uint64_t len,
                   double out[2]) {
  if (!ctx || !a || !b || !table || !out) return invalid("qsb_diag_inner: null argument");
  return diag_inner_exact(ctx, (const double2*)a, table, (const double2*)b, len, out);
}

int qsb_xsum(qsb_ctx* ctx, const double* a, const double* b, uint64_t len, int n_qubits, double out[2]) {
  if (!ctx || !a || !b || !out) return invalid("qsb_xsum: null argument");
  if (n_qubits < 0 || (n_qubits > 0 && (len >> (n_qubits - 1)) < 2))
    return invalid("qsb_xsum: %d qubits do not fit length %llu", n_qubits, (unsigned long long)len);
  return xsum_exact(ctx, (const double2*)a, (const double2*)b, len, n_qubits, out);
}

int qsb_pairwise_level(qsb_ctx* ctx, const double* src, double* dst, uint64_t dst_len) {
  if (!ctx || !src || !dst) return invalid("qsb_pairwise_level: null argument");
  if (!dst_len) return QSB_OK;
  k_pairwise_level<<<grid_for(dst_len, 4), kThreads, 0, ctx->stream>>>(src, dst, dst_len);
  QSB_CHECK_LAUNCH(ctx, "pairwise_level");
  return QSB_OK;
}

}  // extern "C"
