// Native NCCL transport of the sharded qubit swap (dist.py TorchExchanger, non-P2P mode).
//
// The swap is an all-to-all of equal chunks: chunk c (the amplitudes whose top g local
// bits are c) of every shard goes to shard c and lands as its chunk r.  Here it is one
// NCCL group of send/recv pairs issued on the context's own stream, so it is ordered
// after the sweep that produced the data and before the next one with no host round
// trip (the torch.distributed path had to synchronise the context stream, hand the
// buffers to torch's NCCL stream and synchronise again).
//
// libnccl is opened at run time (dlopen "libnccl.so.2": the copy torch already loaded
// when there is one), so libqsb loads on machines without NCCL and the P2P transport
// does not depend on it.  Only the types come from nccl.h.
#include <dlfcn.h>

#include <chrono>
#include <thread>
#include <nccl.h>

#include "common.cuh"

using namespace qsb;

struct qsb_nccl {
  ncclComm_t comm = nullptr;
  qsb_ctx* ctx = nullptr;
  int nranks = 0, rank = 0;
};

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*version)(int*) = nullptr;
  ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*abort)(ncclComm_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = e ? e : "dlopen(libnccl.so.2) failed";
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    a.ok = sym(a.get_unique_id, "ncclGetUniqueId") && sym(a.comm_init_rank, "ncclCommInitRank") &&
           sym(a.comm_destroy, "ncclCommDestroy") && sym(a.group_start, "ncclGroupStart") &&
           sym(a.group_end, "ncclGroupEnd") && sym(a.send, "ncclSend") && sym(a.recv, "ncclRecv") &&
           sym(a.error_string, "ncclGetErrorString") && sym(a.version, "ncclGetVersion") &&
           sym(a.get_async_error, "ncclCommGetAsyncError") && sym(a.abort, "ncclCommAbort");
    if (!a.ok) a.why = "libnccl.so.2 lacks a needed symbol";
  });
  return a;
}

int nccl_fail(ncclResult_t r, const char* what) {
  set_error("%s: %s", what, api().error_string ? api().error_string(r) : "NCCL error");
  return QSB_ECUDA;
}

#define QSB_NCCL(call)                                       \
  do {                                                       \
    ncclResult_t _r = (call);                                \
    if (_r != ncclSuccess) return nccl_fail(_r, #call);      \
  } while (0)

int need_api() {
  const NcclApi& a = api();
  if (!a.ok) return invalid("NCCL is not available: %s", a.why.c_str());
  return QSB_OK;
}

}  // namespace

extern "C" {

int qsb_nccl_version(int* version) {
  if (!version) return invalid("qsb_nccl_version: null argument");
  QSB_TRY(need_api());
  QSB_NCCL(api().version(version));
  return QSB_OK;
}

int qsb_nccl_unique_id(void* id) {
  if (!id) return invalid("qsb_nccl_unique_id: null argument");
  QSB_TRY(need_api());
  ncclUniqueId u;
  QSB_NCCL(api().get_unique_id(&u));
  memcpy(id, &u, sizeof(u));
  return QSB_OK;
}

int qsb_nccl_init(qsb_ctx* ctx, const void* id, int nranks, int rank, qsb_nccl** out) {
  if (!ctx || !id || !out) return invalid("qsb_nccl_init: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return invalid("qsb_nccl_init: rank %d of %d", rank, nranks);
  *out = nullptr;
  QSB_TRY(need_api());
  QSB_CUDA(cudaSetDevice(ctx->device));
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  qsb_nccl* c = new qsb_nccl;
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = api().comm_init_rank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return QSB_OK;
}

// dst chunk c <- shard c's src chunk r, for every c (chunk_amps complex128 amplitudes per
// chunk), on the context stream.  src and dst must not overlap.
int qsb_nccl_all_to_all(qsb_nccl* c, const double* src, double* dst, uint64_t chunk_amps) {
  if (!c || !src || !dst) return invalid("qsb_nccl_all_to_all: null argument");
  QSB_CUDA(cudaSetDevice(c->ctx->device));
  if (!chunk_amps) return QSB_OK;
  const size_t count = (size_t)chunk_amps * 2;  // doubles per chunk
  const NcclApi& a = api();
  QSB_NCCL(a.group_start());
  for (int p = 0; p < c->nranks; ++p) {
    const ncclResult_t rs = a.send(src + (size_t)p * count, count, ncclFloat64, p, c->comm, c->ctx->stream);
    const ncclResult_t rr = rs == ncclSuccess ? a.recv(dst + (size_t)p * count, count, ncclFloat64, p, c->comm,
                                                       c->ctx->stream)
                                              : rs;
    if (rr != ncclSuccess) {
      a.group_end();
      return nccl_fail(rr, "ncclSend/ncclRecv");
    }
  }
  QSB_NCCL(a.group_end());
  return QSB_OK;
}

// Failure detection for the stream-ordered all-to-all: wait for the context stream while
// polling the communicator's asynchronous error; on an NCCL error, or when the stream has
// not finished after timeout_ms (a peer that died mid-swap leaves its partners' receives
// pending forever), abort the communicator -- which releases the stuck kernels -- and
// return an error instead of hanging.  timeout_ms < 0: no timeout.
int qsb_nccl_wait(qsb_nccl* c, int64_t timeout_ms) {
  if (!c) return invalid("qsb_nccl_wait: null argument");
  if (!c->comm) return invalid("qsb_nccl_wait: the communicator was aborted");
  QSB_CUDA(cudaSetDevice(c->ctx->device));
  const NcclApi& a = api();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->ctx->stream);
    if (q == cudaSuccess) return QSB_OK;
    if (q != cudaErrorNotReady) QSB_CUDA(q);
    ncclResult_t ar = ncclSuccess;
    const ncclResult_t r = a.get_async_error(c->comm, &ar);
    const bool failed = r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress);
    const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (failed || (timeout_ms >= 0 && ms > timeout_ms)) {
      a.abort(c->comm);
      c->comm = nullptr;
      if (failed) return nccl_fail(r != ncclSuccess ? r : ar, "NCCL all-to-all (communicator aborted)");
      set_error("NCCL all-to-all did not finish within %lld ms: communicator aborted", (long long)timeout_ms);
      return QSB_ECUDA;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int qsb_nccl_destroy(qsb_nccl* c) {
  if (!c) return QSB_OK;
  int rc = QSB_OK;
  if (c->comm) {
    cudaSetDevice(c->ctx->device);
    const ncclResult_t r = api().comm_destroy(c->comm);
    if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommDestroy");
  }
  delete c;
  return rc;
}

}  // extern "C"
