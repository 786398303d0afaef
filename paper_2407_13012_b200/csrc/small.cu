// Whole-circuit kernel for small registers (n <= 11, N <= 2048 amplitudes).
//
// Below one 4096-amplitude tile the sweep machinery does not apply and the per-op
// path is launch-bound (~1.5-2.6 ms per value_and_grad, one launch per qubit gate and a
// host round trip per reduction).  Here ONE CTA keeps the ket, the bra and the cost
// table in shared memory and runs the whole simulate / <C> / adjoint walk in a single
// launch with the reference's arithmetic: host-computed Rx (c, s) and phase LUTs,
// FMA-free products (numba_impl.py:47-72), qubits in ascending order
// (backend.py:200-207) and neighbour-pair trees over the (zero-padded) 2048-element
// block (numba_impl.py:89-126), xsum per qubit in ascending order
// (numba_impl.py:200-226) -- bit-identical to the numba kernel set for integral tables.
#include <math.h>

#include <vector>

#include "common.cuh"

using namespace qsb;
using namespace qsbd;

namespace {

constexpr int kST = 256;            // threads
constexpr int kSMax = 2048;         // amplitudes (n <= 11)
constexpr int kSPer = kSMax / kST;  // reduction elements per thread (8 consecutive)

struct SmallArgs {
  double2* ket;          // global statevector (in: mode 3; out: the walked ket)
  const double* table;   // f64 table T
  const void* cidx;      // compact index (kind 1: u8, 2: u16) -> LUT entry
  const double2* lut;    // kind 1/2: [2p][nvals] phase factors (forward layers, then inverse)
  const double* rxcs;    // [2p][2] (c, s): forward Rx(-2 beta_i), then inverse Rx(+2 beta_i)
  const double* ang;     // kind 0: [2p] angle scales (forward -gamma_i, inverse +gamma_i)
  double* out;           // [0] <C>, [1..p] d_gamma, [p+1..2p] d_beta
  double plus_amp;
  int n, p, kind, nvals;
  int mode;              // 0 simulate, 1 simulate + <C>, 2 value_and_grad, 3 gradient of the given ket
  int want_value;
};

// Neighbour-pair tree over 2048 elements, thread t holding elements 8t..8t+7:
// 3 register levels, 5 xor-shuffle levels, 3 levels over the 8 warp sums.
__device__ double block_tree(double v[kSPer], double* wsum) {
#pragma unroll
  for (int w = kSPer / 2; w >= 1; w >>= 1)
#pragma unroll
    for (int e = 0; e < w; ++e) v[e] = __dadd_rn(v[2 * e], v[2 * e + 1]);
  double x = v[0];
#pragma unroll
  for (int k = 0; k < 5; ++k) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 1 << k));
  __syncthreads();  // wsum reuse
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  double w8[kST / 32];
#pragma unroll
  for (int e = 0; e < kST / 32; ++e) w8[e] = wsum[e];
#pragma unroll
  for (int w = kST / 64; w >= 1; w >>= 1)
#pragma unroll
    for (int e = 0; e < w; ++e) w8[e] = __dadd_rn(w8[2 * e], w8[2 * e + 1]);
  return w8[0];  // every thread holds the root
}

__device__ __forceinline__ void small_body(const SmallArgs& a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double2* ket = (double2*)smem_raw;
  double2* bra = ket + kSMax;
  double* T = (double*)(bra + kSMax);
  double* wsum = T + kSMax;  // 8 warp partials (x2 for re / im)
  const int n = a.n, p = a.p, N = 1 << n, tid = threadIdx.x;

  for (int i = tid; i < N; i += kST) T[i] = a.table[i];
  if (a.mode == 3) {
    for (int i = tid; i < N; i += kST) ket[i] = a.ket[i];
  } else {
    for (int i = tid; i < N; i += kST) ket[i] = make_double2(a.plus_amp, 0.0);
  }
  __syncthreads();

  // ψ_i *= (cos(ang), sin(ang)), ang = scale * T_i (numba_impl.py:47-51)
  auto phase = [&](double2* v, int layer) {
    for (int i = tid; i < N; i += kST) {
      double2 f;
      if (a.kind == 1) f = a.lut[(size_t)layer * a.nvals + ((const uint8_t*)a.cidx)[i]];
      else if (a.kind == 2) f = a.lut[(size_t)layer * a.nvals + ((const uint16_t*)a.cidx)[i]];
      else {
        double s, c;
        sincos(__dmul_rn(a.ang[layer], T[i]), &s, &c);
        f = make_double2(c, s);
      }
      v[i] = cmul_exact(v[i], f);
    }
    __syncthreads();
  };
  // Rx on qubits 0..n-1 ascending (numba_impl.py:60-72, backend.py:200-207)
  auto rx_layer = [&](double2* v, int layer) {
    const double c = a.rxcs[2 * layer], s = a.rxcs[2 * layer + 1];
    for (int j = 0; j < n; ++j) {
      const int low = (1 << j) - 1, bit = 1 << j;
      for (int k = tid; k < (N >> 1); k += kST) {
        const int i0 = ((k & ~low) << 1) | (k & low), i1 = i0 | bit;
        const double2 t = v[i0], u = v[i1];
        v[i0] = make_double2(__dadd_rn(__dmul_rn(c, t.x), __dmul_rn(s, u.y)), __dadd_rn(__dmul_rn(c, t.y), -__dmul_rn(s, u.x)));
        v[i1] = make_double2(__dadd_rn(__dmul_rn(s, t.y), __dmul_rn(c, u.x)), __dadd_rn(__dmul_rn(c, u.y), -__dmul_rn(s, t.x)));
      }
      __syncthreads();
    }
  };

  if (a.mode != 3) {
    for (int i = 0; i < p; ++i) {
      phase(ket, i);
      rx_layer(ket, i);
    }
  }
  if (a.want_value) {  // T_i * (re^2 + im^2), tree (numba_impl.py:75-79, 114-126)
    double v[kSPer];
#pragma unroll
    for (int e = 0; e < kSPer; ++e) {
      const int i = tid * kSPer + e;
      v[e] = i < N ? __dmul_rn(T[i], norm2_exact(ket[i])) : 0.0;
    }
    const double r = block_tree(v, wsum);
    if (tid == 0) a.out[0] = r;
  }
  if (a.mode >= 2) {
    for (int i = tid; i < N; i += kST) bra[i] = make_double2(__dmul_rn(ket[i].x, T[i]), __dmul_rn(ket[i].y, T[i]));
    __syncthreads();
    for (int L = p - 1; L >= 0; --L) {
      // xsum (numba_impl.py:200-226): per qubit a tree of conj(bra_i) ket_{i^bit}, += in ascending j
      double xre = 0.0, xim = 0.0;
      for (int j = 0; j < n; ++j) {
        double vr[kSPer], vi[kSPer];
#pragma unroll
        for (int e = 0; e < kSPer; ++e) {
          const int i = tid * kSPer + e;
          if (i < N) {
            const double2 pa = bra[i], q = ket[i ^ (1 << j)];
            vr[e] = re_conj_mul_exact(pa, q);
            vi[e] = im_conj_mul_exact(pa, q);
          } else {
            vr[e] = vi[e] = 0.0;
          }
        }
        xre = __dadd_rn(xre, block_tree(vr, wsum));
        xim = __dadd_rn(xim, block_tree(vi, wsum + kST / 32));
      }
      if (tid == 0) a.out[1 + p + L] = -2.0 * xim;
      rx_layer(bra, p + L);
      rx_layer(ket, p + L);
      // <bra|C|ket> (numba_impl.py:173-197): products, then * T
      double vr[kSPer], vi[kSPer];
#pragma unroll
      for (int e = 0; e < kSPer; ++e) {
        const int i = tid * kSPer + e;
        if (i < N) {
          const double2 pa = bra[i], q = ket[i];
          vr[e] = __dmul_rn(re_conj_mul_exact(pa, q), T[i]);
          vi[e] = __dmul_rn(im_conj_mul_exact(pa, q), T[i]);
        } else {
          vr[e] = vi[e] = 0.0;
        }
      }
      block_tree(vr, wsum);
      const double di = block_tree(vi, wsum + kST / 32);
      if (tid == 0) a.out[1 + L] = 2.0 * di;
      phase(bra, p + L);
      phase(ket, p + L);
    }
  }
  for (int i = tid; i < N; i += kST) a.ket[i] = ket[i];
}

__global__ void __launch_bounds__(kST, 1) k_small(const SmallArgs a) { small_body(a); }

// batched: one CTA per (handle, parameters) instance -- the paper's many-small-graphs
// regime (444-graph suite, optimizer restarts) in one launch
__global__ void __launch_bounds__(kST, 1) k_small_batch(const SmallArgs* __restrict__ args) {
  const SmallArgs a = args[blockIdx.x];
  small_body(a);
}

constexpr size_t kSmallSmem = (size_t)kSMax * (16 + 16 + 8) + 2 * (kST / 32) * sizeof(double);

}  // namespace

namespace qsb {

// Host side: LUTs / angles / Rx coefficients for 2p layers (forward, then inverse),
// one launch, one copy back.  mode: 0 simulate, 1 simulate + <C>, 2 value_and_grad,
// 3 gradient of the ket as given.
int small_run(qsb_ctx* ctx, qsb_table* t, double2* ket, int p, const double* gammas, const double* betas, int mode,
              double* value, double* dg, double* db) {
  const int n = t->n;
  if (n > 11) return invalid("internal: small_run needs n <= 11");
  const int L = 2 * (p > 0 ? p : 1);
  std::vector<double> host(4 * L + 1 + 2 * p + 1, 0.0);
  double* rxcs = host.data();          // [L][2]
  double* ang = rxcs + 2 * L;          // [L]
  for (int i = 0; i < p; ++i) {
    const double tf = -2.0 * betas[i], ti = 2.0 * betas[i];  // circuit.py:103, adjoint.py:63-64
    rxcs[2 * i] = cos(tf / 2.0);
    rxcs[2 * i + 1] = sin(tf / 2.0);
    rxcs[2 * (p + i)] = cos(ti / 2.0);
    rxcs[2 * (p + i) + 1] = sin(ti / 2.0);
    ang[i] = -gammas[i];      // forward phase exp(-i g C)
    ang[p + i] = gammas[i];   // inverse phase (adjoint.py:67-68 phase(-gamma))
  }
  if (t->kind != 0) {
    std::vector<double> sc(ang, ang + 2 * p);
    std::vector<double2> ex(2 * p, make_double2(1.0, 0.0));
    if (p > 0) QSB_TRY(prepare_luts(t, sc, ex, true));
  }
  const size_t in_bytes = (size_t)(3 * L) * sizeof(double);
  const size_t out_doubles = 1 + 2 * (size_t)p;
  QSB_TRY(ensure_small(ctx, in_bytes + out_doubles * sizeof(double) + 64));
  double* d_in = (double*)ctx->d_small;
  double* d_out = d_in + 3 * L;
  QSB_CUDA(cudaMemcpyAsync(d_in, host.data(), in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += in_bytes;
  SmallArgs a;
  a.ket = ket;
  a.table = t->values;
  a.cidx = t->cidx;
  a.lut = t->d_lut;
  a.rxcs = d_in;
  a.ang = d_in + 2 * L;
  a.out = d_out;
  a.plus_amp = 1.0 / sqrt((double)(1ull << n));  // numba_impl.py:42
  a.n = n;
  a.p = p;
  a.kind = t->kind;
  a.nvals = t->nvals;
  a.mode = mode;
  a.want_value = value != nullptr;
  const size_t smem = kSmallSmem;
  static PerDevice<cudaError_t> attr;
  QSB_CUDA(attr.get(ctx->device, [&] {
    cudaError_t e = cudaSetDevice(ctx->device);
    return e != cudaSuccess ? e : cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }));
  k_small<<<1, kST, smem, ctx->stream>>>(a);
  QSB_CHECK_LAUNCH(ctx, "small-register circuit");
  if (value || mode >= 2) {
    double* h = ctx->h_small;
    QSB_CUDA(cudaMemcpyAsync(h, d_out, out_doubles * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->d2h_bytes += out_doubles * sizeof(double);
    if (value) *value = h[0];
    if (mode >= 2)
      for (int i = 0; i < p; ++i) {
        dg[i] = h[1 + i];
        db[i] = h[1 + p + i];
      }
  }
  return QSB_OK;
}

}  // namespace qsb

extern "C" {

// Many small registers in one launch (see qsb.h).  Host work per instance: Rx (c, s)
// and phase LUT / angles, all packed into one upload.
int qsb_small_batch(qsb_ctx* ctx, int count, qsb_table* const* tables, double* const* kets, const int* ps,
                    const double* gammas, const double* betas, int mode, double* out) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || count < 0 || (count > 0 && (!tables || !kets || !ps || !gammas || !betas || !out)))
    return invalid("qsb_small_batch: null argument");
  if (mode < 0 || mode > 2) return invalid("qsb_small_batch: mode must be 0 (simulate), 1 (+<C>) or 2 (+gradient)");
  if (count == 0) return QSB_OK;
  // host staging: per instance [rxcs 4p][ang 2p][lut 2p*nvals*2]; outputs 1 + 2p
  std::vector<size_t> off(count + 1, 0), ooff(count + 1, 0), poff(count + 1, 0);
  for (int k = 0; k < count; ++k) {
    const qsb_table* t = tables[k];
    if (!t || !kets[k]) return invalid("qsb_small_batch: instance %d has no table / state", k);
    if (t->n < 1 || t->n > 11) return invalid("qsb_small_batch: instance %d has n=%d (1..11)", k, t->n);
    if (ps[k] < 1) return invalid("qsb_small_batch: instance %d has p=%d", k, ps[k]);
    const size_t nv = t->kind != 0 ? (size_t)t->nvals : 0;
    off[k + 1] = off[k] + 6 * (size_t)ps[k] + 4 * (size_t)ps[k] * nv;
    ooff[k + 1] = ooff[k] + 1 + 2 * (size_t)ps[k];
    poff[k + 1] = poff[k] + (size_t)ps[k];
  }
  std::vector<double> host(off[count]);
  for (int k = 0; k < count; ++k) {
    const qsb_table* t = tables[k];
    const int p = ps[k];
    const double* g = gammas + poff[k];
    const double* b = betas + poff[k];
    double* rxcs = host.data() + off[k];
    double* ang = rxcs + 4 * p;
    double* lut = ang + 2 * p;
    for (int i = 0; i < p; ++i) {
      const double tf = -2.0 * b[i], ti = 2.0 * b[i];
      rxcs[2 * i] = cos(tf / 2.0);
      rxcs[2 * i + 1] = sin(tf / 2.0);
      rxcs[2 * (p + i)] = cos(ti / 2.0);
      rxcs[2 * (p + i) + 1] = sin(ti / 2.0);
      ang[i] = -g[i];
      ang[p + i] = g[i];
    }
    if (t->kind != 0)
      for (int L = 0; L < 2 * p; ++L)
        for (int v = 0; v < t->nvals; ++v) {
          const double an = ang[L] * (t->vmin + (double)v);  // same product as prepare_luts
          lut[2 * ((size_t)L * t->nvals + v)] = cos(an);
          lut[2 * ((size_t)L * t->nvals + v) + 1] = sin(an);
        }
  }
  // device: [staging][outputs][args]
  const size_t stage_b = host.size() * sizeof(double), out_b = ooff[count] * sizeof(double);
  const size_t args_b = (size_t)count * sizeof(SmallArgs);
  QSB_TRY(ensure_small(ctx, stage_b + out_b + args_b + 256));
  double* d_stage = (double*)ctx->d_small;
  double* d_out = d_stage + host.size();
  SmallArgs* d_args = (SmallArgs*)(((uintptr_t)(d_out + ooff[count]) + 15) & ~(uintptr_t)15);
  std::vector<SmallArgs> args(count);
  for (int k = 0; k < count; ++k) {
    const qsb_table* t = tables[k];
    SmallArgs& a = args[k];
    a.ket = (double2*)kets[k];
    a.table = t->values;
    a.cidx = t->cidx;
    a.rxcs = d_stage + off[k];
    a.ang = a.rxcs + 4 * ps[k];
    a.lut = (const double2*)(a.ang + 2 * ps[k]);
    a.out = d_out + ooff[k];
    a.plus_amp = 1.0 / sqrt((double)(1ull << t->n));
    a.n = t->n;
    a.p = ps[k];
    a.kind = t->kind;
    a.nvals = t->nvals;
    a.mode = mode;
    a.want_value = mode >= 1;
  }
  QSB_CUDA(cudaMemcpyAsync(d_stage, host.data(), stage_b, cudaMemcpyHostToDevice, ctx->stream));
  QSB_CUDA(cudaMemcpyAsync(d_args, args.data(), args_b, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += stage_b + args_b;
  static PerDevice<cudaError_t> attr;
  QSB_CUDA(attr.get(ctx->device, [&] {
    cudaError_t e = cudaSetDevice(ctx->device);
    return e != cudaSuccess ? e : cudaFuncSetAttribute(k_small_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
  }));
  k_small_batch<<<count, kST, kSmallSmem, ctx->stream>>>(d_args);
  QSB_CHECK_LAUNCH(ctx, "small-register batch");
  QSB_CUDA(cudaMemcpyAsync(out, d_out, out_b, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->d2h_bytes += out_b;
  return QSB_OK;
}

}  // extern "C"
