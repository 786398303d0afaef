// Shared internals of libqsb: context, error plumbing, complex helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>
#include <mutex>

#include "../../include/qsb.h"

namespace qsb {

// ------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define QSB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::qsb::cuda_fail(_e, #call); \
  } while (0)

#define QSB_CHECK_LAUNCH(ctx, what)                      \
  do {                                                   \
    (ctx)->launches++;                                   \
    cudaError_t _e = cudaGetLastError();                 \
    if (_e != cudaSuccess) return ::qsb::cuda_fail(_e, what); \
  } while (0)

#define QSB_TRY(expr)                                    \
  do {                                                   \
    int _rc = (expr);                                    \
    if (_rc != QSB_OK) return _rc;                       \
  } while (0)

int invalid(const char* fmt, ...);

}  // namespace qsb

// ------------------------------------------------------------ context
struct qsb_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint64_t launches = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic issued by the library
  int last_half = 0;  // the last qsb_simulate_expect (QSB_HALF_OUT) left the upper half unwritten
  // reusable device scratch for reduction partials (grown on demand)
  double* d_scratch = nullptr;
  uint64_t scratch_bytes = 0;
  // sampler scratch (probability-tree levels k0..n + shot outputs), grown on demand and
  // kept: re-allocating ~0.5 GB per draw costs more than the draw itself
  void* d_sample = nullptr;
  uint64_t sample_bytes = 0;
  void* d_shots = nullptr;  // per-shot uniforms / indices / costs
  uint64_t shots_bytes = 0;
  int tree_n = -1;              // the state whose tree d_sample holds (qsb_sample_tree)
  const void* tree_amps = nullptr;
  // pinned host staging for small results
  double* h_small = nullptr;  // 4096 doubles
  // reusable device buffer for small uploads (LUTs, terms)
  void* d_small = nullptr;
  uint64_t small_bytes = 0;
  // forward checkpoints of the adjoint walk (spare HBM, fused.cu run_chain): kept between
  // calls, released when the context is destroyed or an allocation needs the memory
  std::vector<void*> ck;
  uint64_t ck_bytes = 0;
  bool ck_busy = false;  // a walk using them is being enqueued (not released on OOM meanwhile)
  // live per-kernel profiling (qsb_prof_begin/end): CUDA events around each sweep
  bool prof = false;
  struct ProfRec {
    cudaEvent_t a, b;
    int kind;
    double bytes;
  };
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
};

struct qsb_table {
  qsb_ctx* ctx = nullptr;
  int n = 0;
  uint64_t len = 0;
  double* values = nullptr;   // caller-owned fp64 table
  double vmin = 0, vmax = 0;
  int kind = 0;               // 0 fp64/sincos, 1 uint8 idx, 2 uint16 idx
  int nvals = 0;              // number of LUT entries (kind 1/2)
  int sym = 0;                // values[x] == values[len-1-x] for every x (flip-symmetric: Z2 reduction)
  void* cidx = nullptr;       // compact index table (owned)
  double2* d_lut = nullptr;   // phase LUT scratch (owned), up to 65536 entries
  std::vector<double> h_lutbuf;  // host staging
  double2* d_flut = nullptr;  // angle LUTs of an fp64 table (fused.cu FloatLuts), grown on demand
  uint64_t flut_cap = 0;      // entries
};

namespace qsb {
// Kernel function attributes (max dynamic shared memory) and occupancy are per
// device: one-time setup is cached per device ordinal, not per process, so a kernel
// first launched on one GPU still gets its attributes on another.
constexpr int kMaxDevices = 64;
template <class T>
struct PerDevice {
  std::once_flag once[kMaxDevices];
  T val[kMaxDevices];
  template <class F>
  const T& get(int dev, F&& init) {
    const int d = dev < 0 || dev >= kMaxDevices ? 0 : dev;
    std::call_once(once[d], [&] { val[d] = init(); });
    return val[d];
  }
};
// profiling hooks (no-ops unless ctx->prof)
int prof_mark(qsb_ctx* ctx, cudaEvent_t* ev);
int ensure_scratch(qsb_ctx* ctx, uint64_t bytes);
int ensure_small(qsb_ctx* ctx, uint64_t bytes);
int ensure_sample_scratch(qsb_ctx* ctx, uint64_t bytes);
int ensure_shot_scratch(qsb_ctx* ctx, uint64_t bytes);
// up to `want` device buffers of `bytes` each for forward checkpoints, as many as fit in
// free HBM above a margin (QSB_CKPT_MARGIN_GB, default 8; QSB_NO_CKPT=1: none)
int ensure_checkpoints(qsb_ctx* ctx, uint64_t bytes, int want, std::vector<double2*>& out);
void release_checkpoints(qsb_ctx* ctx, bool to_cache = false);
// the large-block cache (ctx.cu): equal-size reuse of multi-GiB buffers
void* big_take(int device, uint64_t bytes);
bool big_put(int device, void* p, uint64_t bytes);
void big_release(int device);
// cudaMalloc that, when the device is full, gives the large-block cache back and retries
inline cudaError_t dev_malloc(void** p, size_t bytes, int device) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    big_release(device);
    e = cudaMalloc(p, bytes);
  }
  return e;
}
// the walk that ensure_checkpoints handed buffers to has enqueued its last use of them
void checkpoints_done(qsb_ctx* ctx);
// build (cos, sin) of (sign * gamma * v) for v = vmin + k, k < nvals, with host libm
// (the same values Python's math.cos/sin and numba give) and upload to t->d_lut.
int upload_phase_lut(qsb_table* t, double ang_scale, double2 extra_scale, bool exact);
// per-call phase LUTs for compact tables: LUT k = t->d_lut + k * nvals holds (cos, sin)
// of ang_scales[k] * v (times extras[k] unless exact), v = vmin + index (fused.cu)
int prepare_luts(qsb_table* t, const std::vector<double>& ang_scales, const std::vector<double2>& extras, bool exact);
}  // namespace qsb

// ------------------------------------------------------------ device helpers
namespace qsbd {

__device__ __forceinline__ double2 cmul_exact(double2 a, double2 b) {
  // (ar*br - ai*bi, ar*bi + ai*br), each product rounded separately (numba complex *)
  return make_double2(__dadd_rn(__dmul_rn(a.x, b.x), -__dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cmul_fast(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <bool EXACT>
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  if constexpr (EXACT) return cmul_exact(a, b); else return cmul_fast(a, b);
}
// |a|^2 as numba computes it: a.real*a.real + a.imag*a.imag, no contraction
__device__ __forceinline__ double norm2_exact(double2 a) {
  return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}
// Im(conj(a) * b) and Re(conj(a) * b) in real arithmetic (numba_impl.py:159-160)
__device__ __forceinline__ double im_conj_mul_exact(double2 a, double2 b) {
  return __dadd_rn(__dmul_rn(a.x, b.y), -__dmul_rn(a.y, b.x));
}
__device__ __forceinline__ double re_conj_mul_exact(double2 a, double2 b) {
  return __dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
}

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_plain(const double2* p) { return *p; }
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace qsbd
