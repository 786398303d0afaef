// Context, memory and error plumbing of libqsb (the C ABI in include/qsb.h).
#include <stdarg.h>
#include <math.h>
#include <string.h>

#include <stdlib.h>

#include <map>
#include <unordered_map>
#include <unordered_set>

#include "common.cuh"

namespace {
thread_local char g_err[1024] = "";
}

namespace qsb {

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  if (e == cudaErrorMemoryAllocation) return QSB_ENOMEM;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorInvalidDevice)
    return QSB_ENODEV;
  return QSB_ECUDA;
}

int invalid(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return QSB_EINVAL;
}

int ensure_scratch(qsb_ctx* ctx, uint64_t bytes) {
  if (bytes <= ctx->scratch_bytes) return QSB_OK;
  if (ctx->d_scratch) {
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    QSB_CUDA(cudaFree(ctx->d_scratch));
    ctx->d_scratch = nullptr;
    ctx->scratch_bytes = 0;
  }
  uint64_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
  QSB_CUDA(dev_malloc((void**)&ctx->d_scratch, want, ctx->device));
  ctx->scratch_bytes = want;
  return QSB_OK;
}

int ensure_sample_scratch(qsb_ctx* ctx, uint64_t bytes) {
  if (bytes <= ctx->sample_bytes) return QSB_OK;
  if (ctx->d_sample) {
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    QSB_CUDA(cudaFree(ctx->d_sample));
    ctx->d_sample = nullptr;
    ctx->sample_bytes = 0;
  }
  ctx->tree_n = -1;
  cudaError_t e = cudaMalloc(&ctx->d_sample, bytes);
  if (e == cudaErrorMemoryAllocation) {  // cached large blocks may be in the way
    cudaGetLastError();
    big_release(ctx->device);
    e = cudaMalloc(&ctx->d_sample, bytes);
  }
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return ::qsb::cuda_fail(e, "sampler scratch");
  }
  QSB_CUDA(e);
  ctx->sample_bytes = bytes;
  return QSB_OK;
}

int ensure_shot_scratch(qsb_ctx* ctx, uint64_t bytes) {
  if (bytes <= ctx->shots_bytes) return QSB_OK;
  if (ctx->d_shots) {
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    QSB_CUDA(cudaFree(ctx->d_shots));
    ctx->d_shots = nullptr;
    ctx->shots_bytes = 0;
  }
  QSB_CUDA(dev_malloc((void**)&ctx->d_shots, bytes, ctx->device));
  ctx->shots_bytes = bytes;
  return QSB_OK;
}

int ensure_small(qsb_ctx* ctx, uint64_t bytes) {
  if (bytes <= ctx->small_bytes) return QSB_OK;
  if (ctx->d_small) {
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    QSB_CUDA(cudaFree(ctx->d_small));
    ctx->d_small = nullptr;
    ctx->small_bytes = 0;
  }
  uint64_t want = bytes < (1u << 16) ? (1u << 16) : bytes;
  QSB_CUDA(dev_malloc((void**)&ctx->d_small, want, ctx->device));
  ctx->small_bytes = want;
  return QSB_OK;
}

// Large-block cache.  cudaMalloc / cudaFree of multi-GiB buffers cost milliseconds per
// GiB (page-table work; cudaFree also synchronises the device), which made
// create_handle / close and every first gradient of a fresh handle at n >= 26 cost
// more than the E+grad itself.  Buffers above the stream-ordered pool's size (qsb_alloc
// > 1 GiB) and forward checkpoints go back to a per-device cache on free (after their
// stream has finished with them) and are handed out again for an equal size; an
// allocation that runs out of memory, or a checkpoint set that needs memory the cache
// holds, releases the cache first.  QSB_NO_BIGCACHE=1 disables it.
namespace {
constexpr uint64_t kBigKeep = 96ull << 30;
std::mutex g_big_mu;
std::multimap<uint64_t, void*> g_big[qsb::kMaxDevices];
uint64_t g_big_bytes[qsb::kMaxDevices] = {};

bool big_cache_enabled() {
  const char* e = getenv("QSB_NO_BIGCACHE");
  return !(e && atoi(e));
}
}  // namespace

// a cached block of exactly `bytes`, or nullptr
void* big_take(int device, uint64_t bytes) {
  if (!big_cache_enabled()) return nullptr;
  std::lock_guard<std::mutex> g(g_big_mu);
  auto it = g_big[device].find(bytes);
  if (it == g_big[device].end()) return nullptr;
  void* p = it->second;
  g_big[device].erase(it);
  g_big_bytes[device] -= bytes;
  return p;
}

// keep a block whose last uses have completed; false: the caller frees it
bool big_put(int device, void* p, uint64_t bytes) {
  if (!big_cache_enabled()) return false;
  std::lock_guard<std::mutex> g(g_big_mu);
  if (g_big_bytes[device] + bytes > kBigKeep) return false;
  g_big[device].emplace(bytes, p);
  g_big_bytes[device] += bytes;
  return true;
}

void big_release(int device) {
  std::multimap<uint64_t, void*> blocks;
  {
    std::lock_guard<std::mutex> g(g_big_mu);
    blocks.swap(g_big[device]);
    g_big_bytes[device] = 0;
  }
  if (blocks.empty()) return;
  cudaSetDevice(device);
  for (auto& kv : blocks) cudaFree(kv.second);
}

// free cached blocks (largest first) until at least `need` bytes are free on the device
// or the cache is empty -- cudaFree of multi-GiB blocks costs tens of ms each, so a size
// change releases only what the new allocations need
void big_release_until(int device, uint64_t need) {
  cudaSetDevice(device);
  for (;;) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || fr >= need) return;
    void* p = nullptr;
    {
      std::lock_guard<std::mutex> g(g_big_mu);
      if (g_big[device].empty()) return;
      auto it = std::prev(g_big[device].end());
      p = it->second;
      g_big_bytes[device] -= it->first;
      g_big[device].erase(it);
    }
    cudaFree(p);
  }
}

// Forward checkpoints.  Contexts holding them are registered so an allocation that runs
// out of memory (on any thread) can take the memory back (release_all_checkpoints).
// g_ck_mu guards every context's ck / ck_bytes / ck_busy; a context whose walk is being
// enqueued (ck_busy, from ensure_checkpoints to checkpoints_done) keeps its buffers.
namespace {
std::mutex g_ck_mu;
std::unordered_set<qsb_ctx*> g_ck_ctxs;

void release_locked(qsb_ctx* ctx, bool to_cache = false) {  // g_ck_mu held
  if (ctx->ck.empty()) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);  // kernels already enqueued may still read them
  for (void* p : ctx->ck)
    if (!to_cache || !qsb::big_put(ctx->device, p, ctx->ck_bytes)) cudaFree(p);
  ctx->ck.clear();
  ctx->ck_bytes = 0;
  g_ck_ctxs.erase(ctx);
}
}  // namespace

void release_checkpoints(qsb_ctx* ctx, bool to_cache) {
  std::lock_guard<std::mutex> g(g_ck_mu);
  release_locked(ctx, to_cache);
}

void release_all_checkpoints() {
  std::lock_guard<std::mutex> g(g_ck_mu);
  std::vector<qsb_ctx*> all(g_ck_ctxs.begin(), g_ck_ctxs.end());
  for (qsb_ctx* c : all)
    if (!c->ck_busy) release_locked(c);
}

int ensure_checkpoints(qsb_ctx* ctx, uint64_t bytes, int want, std::vector<double2*>& out) {
  out.clear();
  const char* off = getenv("QSB_NO_CKPT");
  if ((off && atoi(off)) || want <= 0) return QSB_OK;
  std::lock_guard<std::mutex> g(g_ck_mu);
  if (ctx->ck_bytes != bytes) release_locked(ctx);
  while ((int)ctx->ck.size() < want) {  // equal-size blocks from the large-block cache
    void* p = big_take(ctx->device, bytes);
    if (!p) break;
    ctx->ck.push_back(p);
  }
  if ((int)ctx->ck.size() < want) {
    const char* m = getenv("QSB_CKPT_MARGIN_GB");
    const uint64_t margin = (uint64_t)(m ? atof(m) : 8.0) << 30;
    // cached blocks of other sizes give back only what the missing checkpoints need
    big_release_until(ctx->device, margin + bytes * (uint64_t)(want - (int)ctx->ck.size()) + bytes);
    size_t fr = 0, tot = 0;
    QSB_CUDA(cudaMemGetInfo(&fr, &tot));
    while ((int)ctx->ck.size() < want && fr > margin + bytes) {
      void* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        break;
      }
      ctx->ck.push_back(p);
      fr -= bytes;
    }
  }
  ctx->ck_bytes = ctx->ck.empty() ? 0 : bytes;
  if (!ctx->ck.empty()) g_ck_ctxs.insert(ctx);
  for (int i = 0; i < want && i < (int)ctx->ck.size(); ++i) out.push_back((double2*)ctx->ck[i]);
  ctx->ck_busy = !out.empty();
  return QSB_OK;
}

void checkpoints_done(qsb_ctx* ctx) {
  std::lock_guard<std::mutex> g(g_ck_mu);
  ctx->ck_busy = false;
}

int prof_mark(qsb_ctx* ctx, cudaEvent_t* ev) {
  if (ctx->prof_used == ctx->prof_pool.size()) {
    cudaEvent_t e;
    QSB_CUDA(cudaEventCreate(&e));
    ctx->prof_pool.push_back(e);
  }
  *ev = ctx->prof_pool[ctx->prof_used++];
  QSB_CUDA(cudaEventRecord(*ev, ctx->stream));
  return QSB_OK;
}

}  // namespace qsb

using namespace qsb;

extern "C" {

const char* qsb_last_error(void) { return g_err; }
int qsb_abi_version(void) { return 1; }

int qsb_device_count(int* out) {
  if (!out) return invalid("qsb_device_count: null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = n;
  return QSB_OK;
}

// Context pool: creating a context costs 5-30 ms (stream, events, pinned staging,
// device queries) -- more than a whole small-register E+grad.  Destroyed contexts go
// back to a per-device free list with their stream, events, pinned buffer and small
// scratch (the sampler's large scratch is released) and qsb_ctx_create reuses them.
namespace {
constexpr size_t kPoolCap = 32;
std::mutex g_pool_mu;
std::vector<qsb_ctx*> g_pool[qsb::kMaxDevices];

struct DevInfo {
  cudaError_t err;
  int major, sms;
};
qsb::PerDevice<DevInfo> g_devinfo;

void reset_for_reuse(qsb_ctx* ctx) {
  ctx->launches = 0;
  ctx->h2d_bytes = ctx->d2h_bytes = 0;
  ctx->last_half = 0;
  ctx->tree_n = -1;
  ctx->tree_amps = nullptr;
  ctx->prof = false;
  ctx->prof_recs.clear();
  ctx->prof_used = 0;
}
}  // namespace

int qsb_ctx_create(int device, qsb_ctx** out) {
  if (!out) return invalid("qsb_ctx_create: null out");
  *out = nullptr;
  if (device < 0 || device >= kMaxDevices) return invalid("qsb_ctx_create: device %d out of range", device);
  QSB_CUDA(cudaSetDevice(device));
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pool[device].empty()) {
      qsb_ctx* ctx = g_pool[device].back();
      g_pool[device].pop_back();
      reset_for_reuse(ctx);
      *out = ctx;
      return QSB_OK;
    }
  }
  const DevInfo& info = g_devinfo.get(device, [&] {
    DevInfo d{cudaSuccess, 0, 0};
    d.err = cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, device);
    if (d.err == cudaSuccess) d.err = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device);
    return d;
  });
  QSB_CUDA(info.err);
  if (info.major < 10) return invalid("device %d is sm_%dx; libqsb is built for sm_100a (B200)", device, info.major);
  qsb_ctx* ctx = new qsb_ctx();
  ctx->device = device;
  ctx->num_sms = info.sms;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_small, 4096 * sizeof(double));
  if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "context setup"); }
  *out = ctx;
  return QSB_OK;
}

static void destroy_now(qsb_ctx* ctx) {
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  if (ctx->d_small) cudaFree(ctx->d_small);
  if (ctx->d_sample) cudaFree(ctx->d_sample);
  if (ctx->d_shots) cudaFree(ctx->d_shots);
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int qsb_ctx_destroy(qsb_ctx* ctx) {
  if (!ctx) return QSB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  release_checkpoints(ctx, true);  // into the large-block cache (the next handle's walk)
  // the sampler's scratch is sized by the largest state drawn (0.5 GB at n=30): release it
  if (ctx->d_sample) cudaFree(ctx->d_sample);
  if (ctx->d_shots) cudaFree(ctx->d_shots);
  ctx->d_sample = ctx->d_shots = nullptr;
  ctx->sample_bytes = ctx->shots_bytes = 0;
  if (ctx->scratch_bytes > (64u << 20)) {
    cudaFree(ctx->d_scratch);
    ctx->d_scratch = nullptr;
    ctx->scratch_bytes = 0;
  }
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (g_pool[ctx->device].size() < kPoolCap) {
      g_pool[ctx->device].push_back(ctx);
      return QSB_OK;
    }
  }
  destroy_now(ctx);
  return QSB_OK;
}

int qsb_ctx_sync(qsb_ctx* ctx) {
  if (!ctx) return invalid("null context");
  QSB_CUDA(cudaSetDevice(ctx->device));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

int qsb_ctx_device(qsb_ctx* ctx, int* device) {
  if (!ctx || !device) return invalid("null argument");
  *device = ctx->device;
  return QSB_OK;
}

int qsb_ctx_info(qsb_ctx* ctx, int* num_sms, uint64_t* free_bytes, uint64_t* total_bytes) {
  if (!ctx) return invalid("null context");
  QSB_CUDA(cudaSetDevice(ctx->device));
  size_t f = 0, t = 0;
  QSB_CUDA(cudaMemGetInfo(&f, &t));
  if (num_sms) *num_sms = ctx->num_sms;
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = t;
  return QSB_OK;
}

int qsb_timer_start(qsb_ctx* ctx) {
  if (!ctx) return invalid("null context");
  QSB_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  return QSB_OK;
}

int qsb_timer_stop(qsb_ctx* ctx, double* ms) {
  if (!ctx || !ms) return invalid("null argument");
  QSB_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  QSB_CUDA(cudaEventSynchronize(ctx->ev1));
  float f = 0;
  QSB_CUDA(cudaEventElapsedTime(&f, ctx->ev0, ctx->ev1));
  *ms = f;
  return QSB_OK;
}

int qsb_prof_begin(qsb_ctx* ctx) {
  if (!ctx) return invalid("null context");
  ctx->prof = true;
  ctx->prof_recs.clear();
  ctx->prof_used = 0;
  return QSB_OK;
}

// out[3*k + 0..2] = launches, total ms, algorithmic bytes for kernel kind k =
// (mode * 2 + nv - 1) * 2 + (B window ? 1 : 0) (mode: 0 plain, 1 merged, 2 bridge);
// nkinds entries are written.
int qsb_prof_end(qsb_ctx* ctx, double* out, int nkinds) {
  if (!ctx || !out) return invalid("null argument");
  ctx->prof = false;
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < 3 * nkinds; ++k) out[k] = 0.0;
  for (const auto& r : ctx->prof_recs) {
    if (r.kind < 0 || r.kind >= nkinds) continue;
    float ms = 0;
    QSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    out[3 * r.kind] += 1.0;
    out[3 * r.kind + 1] += ms;
    out[3 * r.kind + 2] += r.bytes;
  }
  ctx->prof_recs.clear();
  ctx->prof_used = 0;
  return QSB_OK;
}

int qsb_ctx_xfer(qsb_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
  if (!ctx) return invalid("null context");
  if (h2d) *h2d = ctx->h2d_bytes;
  if (d2h) *d2h = ctx->d2h_bytes;
  return QSB_OK;
}

int qsb_ctx_launches(qsb_ctx* ctx, uint64_t* out) {
  if (!ctx || !out) return invalid("null argument");
  *out = ctx->launches;
  return QSB_OK;
}

}  // extern "C"

// Device memory.  cudaMalloc / cudaFree cost milliseconds each (cudaFree synchronises
// the device) -- per handle that is more than a small register's whole E+grad -- so
// buffers up to 1 GiB come from the device's stream-ordered pool (cudaMallocAsync on
// the context's stream, cudaFreeAsync back to it, up to 8 GiB kept cached); larger ones
// and CUDA-IPC-exported shard buffers (qsb_alloc_ipc) use cudaMalloc.
namespace {
constexpr uint64_t kPooledMax = 1ull << 30;
constexpr uint64_t kPoolKeep = 8ull << 30;
std::mutex g_alloc_mu;
std::unordered_set<void*> g_pooled;
qsb::PerDevice<cudaError_t> g_poolcfg;

bool pool_enabled() {
  const char* e = getenv("QSB_NO_MEMPOOL");
  return !(e && atoi(e));
}

std::unordered_map<void*, uint64_t> g_big_live;  // qsb_alloc blocks > kPooledMax (cacheable), guarded by g_alloc_mu

int plain_alloc(qsb_ctx* ctx, uint64_t bytes, void** dptr) {
  cudaError_t e = cudaMalloc(dptr, bytes ? bytes : 16);
  if (e == cudaErrorMemoryAllocation) {  // checkpoints / cached blocks / pool memory may be in the way
    cudaGetLastError();
    qsb::release_all_checkpoints();
    qsb::big_release(ctx->device);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
    }
    e = cudaMalloc(dptr, bytes ? bytes : 16);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %llu bytes failed (%s)", (unsigned long long)bytes, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? QSB_ENOMEM : QSB_ECUDA;
  }
  return QSB_OK;
}
}  // namespace

extern "C" {

int qsb_alloc(qsb_ctx* ctx, uint64_t bytes, void** dptr) {
  if (!ctx || !dptr) return invalid("null argument");
  QSB_CUDA(cudaSetDevice(ctx->device));
  *dptr = nullptr;
  if (bytes <= kPooledMax && pool_enabled()) {
    const cudaError_t cfg = g_poolcfg.get(ctx->device, [&] {
      cudaMemPool_t pool;
      cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, ctx->device);
      uint64_t keep = kPoolKeep;
      if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      return e;
    });
    if (cfg == cudaSuccess) {
      cudaError_t e = cudaMallocAsync(dptr, bytes ? bytes : 16, ctx->stream);
      if (e == cudaSuccess) {
        std::lock_guard<std::mutex> g(g_alloc_mu);
        g_pooled.insert(*dptr);
        return QSB_OK;
      }
      cudaGetLastError();  // fall through to cudaMalloc
      *dptr = nullptr;
    }
  }
  if (bytes > kPooledMax) {
    void* p = qsb::big_take(ctx->device, bytes);
    if (!p) QSB_TRY(plain_alloc(ctx, bytes, &p));
    std::lock_guard<std::mutex> g(g_alloc_mu);
    g_big_live[p] = bytes;
    *dptr = p;
    return QSB_OK;
  }
  return plain_alloc(ctx, bytes, dptr);
}

int qsb_alloc_ipc(qsb_ctx* ctx, uint64_t bytes, void** dptr) {
  if (!ctx || !dptr) return invalid("null argument");
  QSB_CUDA(cudaSetDevice(ctx->device));
  *dptr = nullptr;
  return plain_alloc(ctx, bytes, dptr);
}

// ctx may be NULL (its context already destroyed): cudaFree synchronises the
// device implicitly, so queued work on any stream has finished with the buffer.
int qsb_free(qsb_ctx* ctx, void* dptr) {
  if (!dptr) return QSB_OK;
  bool pooled;
  uint64_t big = 0;
  {
    std::lock_guard<std::mutex> g(g_alloc_mu);
    pooled = g_pooled.erase(dptr) > 0;
    auto it = g_big_live.find(dptr);
    if (it != g_big_live.end()) {
      big = it->second;
      g_big_live.erase(it);
    }
  }
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));
  if (pooled && ctx) {
    QSB_CUDA(cudaFreeAsync(dptr, ctx->stream));  // stream-ordered after its uses
    return QSB_OK;
  }
  if (big) {  // the buffer's uses are done once its stream (or, with no context, the device) is
    int dev = 0;
    if (ctx) {
      dev = ctx->device;
      QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      cudaPointerAttributes at;
      QSB_CUDA(cudaPointerGetAttributes(&at, dptr));
      dev = at.device;
      QSB_CUDA(cudaSetDevice(dev));
      QSB_CUDA(cudaDeviceSynchronize());
    }
    if (qsb::big_put(dev, dptr, big)) return QSB_OK;
  }
  QSB_CUDA(cudaFree(dptr));
  return QSB_OK;
}

int qsb_release_cached_memory(int device) {
  if (device < 0 || device >= qsb::kMaxDevices) return invalid("qsb_release_cached_memory: device %d", device);
  QSB_CUDA(cudaSetDevice(device));
  qsb::release_all_checkpoints();
  qsb::big_release(device);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    QSB_CUDA(cudaDeviceSynchronize());
    QSB_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  return QSB_OK;
}

// CUDA IPC for the sharded walk's fused qubit swap: a shard's spare buffers are exported
// (64-byte handles, exchanged by the host over torch.distributed) and opened by every
// peer process, whose swap-store kernels then write straight into them over NVLink.
int qsb_ipc_handle(qsb_ctx* ctx, const void* dptr, void* handle64) {
  if (!ctx || !dptr || !handle64) return invalid("qsb_ipc_handle: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  QSB_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  QSB_CUDA(cudaIpcGetMemHandle(&h, (void*)dptr));
  memcpy(handle64, &h, 64);
  return QSB_OK;
}

int qsb_ipc_open(qsb_ctx* ctx, const void* handle64, void** dptr) {
  if (!ctx || !handle64 || !dptr) return invalid("qsb_ipc_open: null argument");
  QSB_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  QSB_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return QSB_OK;
}

int qsb_ipc_close(qsb_ctx* ctx, void* dptr) {
  if (!ctx) return invalid("qsb_ipc_close: null context");
  if (!dptr) return QSB_OK;
  QSB_CUDA(cudaSetDevice(ctx->device));
  QSB_CUDA(cudaIpcCloseMemHandle(dptr));
  return QSB_OK;
}

// device-wide completion: the stores of this process's kernels (including peer stores
// over NVLink) are complete and visible once this returns
int qsb_device_sync(qsb_ctx* ctx) {
  if (!ctx) return invalid("qsb_device_sync: null context");
  QSB_CUDA(cudaSetDevice(ctx->device));
  QSB_CUDA(cudaDeviceSynchronize());
  return QSB_OK;
}

int qsb_h2d(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return invalid("null context");
  if (!bytes) return QSB_OK;
  ctx->h2d_bytes += bytes;
  QSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

int qsb_d2h(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return invalid("null context");
  if (!bytes) return QSB_OK;
  ctx->d2h_bytes += bytes;
  QSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

int qsb_h2d_async(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return invalid("null context");
  if (!bytes) return QSB_OK;
  ctx->h2d_bytes += bytes;
  QSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return QSB_OK;
}

int qsb_d2h_async(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return invalid("null context");
  if (!bytes) return QSB_OK;
  ctx->d2h_bytes += bytes;
  QSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return QSB_OK;
}

int qsb_d2d(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  if (!ctx) return invalid("null context");
  if (!bytes) return QSB_OK;
  QSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return QSB_OK;
}

int qsb_host_alloc(uint64_t bytes, void** hptr) {
  if (!hptr) return invalid("null argument");
  QSB_CUDA(cudaMallocHost(hptr, bytes ? bytes : 16));
  return QSB_OK;
}

int qsb_host_free(void* hptr) {
  if (hptr) QSB_CUDA(cudaFreeHost(hptr));
  return QSB_OK;
}

}  // extern "C"
