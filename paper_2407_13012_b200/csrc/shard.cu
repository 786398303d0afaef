// Sharded-statevector data movement outside the fused sweeps (dist.py).
//
// The window chain fuses the qubit swap (layout A <-> B) into the stores of the A
// visit.  Every other place a swap is needed -- a draw after an odd number of
// layers, the exact-mode per-position schedule, shards with fewer than 21 local
// qubits -- runs this standalone all-to-all: chunk c (the amplitudes whose top g
// local bits are c) of this shard goes to shard c, landing as its chunk r.  The
// destinations are plain device pointers, so the same kernel serves virtual shards
// (one GPU) and CUDA-IPC-mapped peer buffers (one process per GPU: the stores cross
// NVLink/NVSwitch; the caller completes the swap with qsb_device_sync + a barrier).
#include "common.cuh"

using namespace qsb;

namespace {

constexpr int kMaxChunks = 8;  // G <= 8 shards
constexpr int kThreads = 512;

struct ScatterArgs {
  const double2* src;
  double2* dst[kMaxChunks];
  uint64_t chunk;    // amplitudes per chunk
  uint64_t dst_off;  // amplitude offset of this shard's chunk in every destination
  int nchunks;
};

// One launch moves all chunks.  A CTA copies 8 contiguous 16-byte amplitudes per
// thread per step (4096 amplitudes = 64 KB per CTA step, all loads issued before the
// stores), so each warp writes whole 512-byte runs to one peer -- full NVLink packets.
__global__ void __launch_bounds__(kThreads) k_scatter_chunks(const __grid_constant__ ScatterArgs a) {
  constexpr int kPer = 8;
  constexpr uint64_t kStep = (uint64_t)kThreads * kPer;
  const uint64_t per_chunk_steps = (a.chunk + kStep - 1) / kStep;
  const uint64_t total = per_chunk_steps * (uint64_t)a.nchunks;
  for (uint64_t s = blockIdx.x; s < total; s += gridDim.x) {
    const int c = (int)(s / per_chunk_steps);
    const uint64_t o = (s % per_chunk_steps) * kStep;
    const double2* src = a.src + (uint64_t)c * a.chunk + o;
    double2* dst = a.dst[c] + a.dst_off + o;
    double2 v[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const uint64_t i = (uint64_t)e * kThreads + threadIdx.x;
      if (o + i < a.chunk) v[e] = qsbd::ld_stream(src + i);
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const uint64_t i = (uint64_t)e * kThreads + threadIdx.x;
      if (o + i < a.chunk) qsbd::st_stream(dst + i, v[e]);
    }
  }
}

__global__ void k_state_mirror(double2* amps, uint64_t half) {
  for (uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; y < half; y += (uint64_t)gridDim.x * blockDim.x)
    amps[half + y] = qsbd::ld_stream(amps + (half - 1 - y));
}

__global__ void k_fill_const(double2* amps, uint64_t len, double re, double im) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x)
    amps[i] = make_double2(re, im);
}

}  // namespace

extern "C" {

int qsb_scatter_chunks(qsb_ctx* ctx, const double* src, uint64_t chunk_amps, int nchunks, void* const* dsts,
                       uint64_t dst_off_amps) {
  if (!ctx || !src || !dsts) return invalid("qsb_scatter_chunks: null argument");
  if (nchunks < 1 || nchunks > kMaxChunks) return invalid("qsb_scatter_chunks: %d chunks (1..%d)", nchunks, kMaxChunks);
  QSB_CUDA(cudaSetDevice(ctx->device));
  if (!chunk_amps) return QSB_OK;
  ScatterArgs a{};
  a.src = (const double2*)src;
  for (int c = 0; c < nchunks; ++c) {
    if (!dsts[c]) return invalid("qsb_scatter_chunks: null destination %d", c);
    a.dst[c] = (double2*)dsts[c];
  }
  a.chunk = chunk_amps;
  a.dst_off = dst_off_amps;
  a.nchunks = nchunks;
  const uint64_t steps = ((chunk_amps + 4095) / 4096) * (uint64_t)nchunks;
  const uint64_t want = (uint64_t)ctx->num_sms * 4;
  const unsigned grid = (unsigned)(steps < want ? steps : want);
  k_scatter_chunks<<<grid, kThreads, 0, ctx->stream>>>(a);
  QSB_CHECK_LAUNCH(ctx, "scatter_chunks");
  return QSB_OK;
}

int qsb_fill_const(qsb_ctx* ctx, double* amps, uint64_t len, double re, double im) {
  if (!ctx || !amps) return invalid("qsb_fill_const: null argument");
  QSB_CUDA(cudaSetDevice(ctx->device));
  if (!len) return QSB_OK;
  uint64_t blocks = (len + 1023) / 1024;
  if (blocks > (uint64_t)ctx->num_sms * 16) blocks = (uint64_t)ctx->num_sms * 16;
  k_fill_const<<<(unsigned)blocks, 256, 0, ctx->stream>>>((double2*)amps, len, re, im);
  QSB_CHECK_LAUNCH(ctx, "fill_const");
  return QSB_OK;
}

int qsb_state_mirror(qsb_ctx* ctx, double* amps, int n) {
  if (!ctx || !amps) return invalid("qsb_state_mirror: null argument");
  if (n < 1 || n > 62) return invalid("qsb_state_mirror: n=%d out of range", n);
  QSB_CUDA(cudaSetDevice(ctx->device));
  const uint64_t half = 1ull << (n - 1);
  uint64_t blocks = (half + 1023) / 1024;
  if (blocks > (uint64_t)ctx->num_sms * 16) blocks = (uint64_t)ctx->num_sms * 16;
  k_state_mirror<<<(unsigned)blocks, 256, 0, ctx->stream>>>((double2*)amps, half);
  QSB_CHECK_LAUNCH(ctx, "state_mirror");
  return QSB_OK;
}

int qsb_ctx_last_half(qsb_ctx* ctx, int* half) {
  if (!ctx || !half) return invalid("qsb_ctx_last_half: null argument");
  *half = ctx->last_half;
  return QSB_OK;
}

int qsb_table_symmetric(qsb_table* t, int* sym) {
  if (!t || !sym) return invalid("qsb_table_symmetric: null argument");
  *sym = t->sym;
  return QSB_OK;
}

int qsb_table_detach_values(qsb_table* t) {
  if (!t) return invalid("qsb_table_detach_values: null table");
  if (t->kind == 0) return invalid("qsb_table_detach_values: an fp64 table has no compact index to fall back on");
  t->values = nullptr;
  return QSB_OK;
}

}  // extern "C"
