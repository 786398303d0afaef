/*
 * qsb.h — C ABI of the B200 QAOA statevector backend ("qsb").
 *
 * This is the drop-in boundary for the reference's kernel-set plugin seam:
 * `qaoasim.kernels.get(name)` returns a module exposing 14 data-parallel
 * functions over 2^n arrays (/root/reference/pkg/src/qaoasim/kernels/__init__.py:47-61,
 * numba_impl.py:247-260).  Every such function has a `qsb_*` counterpart here
 * operating on DEVICE pointers, plus the allocation hooks that backend.py
 * performs with np.empty today (backend.py:133,150,165,264,268) and the fused
 * entry points the fast path uses (simulate / value_and_grad / sample).
 *
 * Conventions
 *   - amplitudes are complex128 interleaved (re, im) = double[2*len]; tables are f64.
 *   - every function returns an int status (QSB_OK == 0); on failure a
 *     thread-local message is available from qsb_last_error().  The Python
 *     wrapper maps QSB_ENOMEM -> ResourceError, QSB_EINVAL -> ContractViolation,
 *     anything else -> RuntimeError (errors.py:4-19 of the reference).
 *   - all launches go on the context's own CUDA stream; functions that return
 *     a scalar synchronise that stream only.  Distinct contexts may be used
 *     from distinct host threads concurrently.
 *   - no torch types, no C++ types: plain pointers and sizes.
 */
#ifndef QSB_H
#define QSB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_OK 0
#define QSB_EINVAL 1
#define QSB_ENOMEM 2
#define QSB_ECUDA 3
#define QSB_ENODEV 4

/* flags for the fused entry points */
#define QSB_EXACT 1u      /* FMA-free arithmetic + ascending qubit order: bit-identical
                             to the numba kernel set (numba_impl.py:47-72) */
#define QSB_FROM_PLUS 2u  /* (simulate) start from |+>, the input state is not read */
#define QSB_HALF_OUT 4u   /* (simulate) a Z2-reduced run may leave the upper half of amps
                             unwritten (psi(2^(n-1)+y) = psi(2^(n-1)-1-y)); qsb_ctx_last_half
                             reports it, qsb_state_mirror writes it */

/* fused-op flags of qsb_layer_sweeps (the sweep kernel's SweepFlags) */
#define QSB_SW_PLUS 1u           /* input is |+> (not read) */
#define QSB_SW_PRE_PHASE 2u      /* multiply by exp(i * phase_scale * C) before the gates */
#define QSB_SW_BRA_FROM_KET 4u   /* nv=2: bra = C * ket (bra not read) */
#define QSB_SW_PRE_DINNER 8u     /* nv=2: sums[1] += Im <bra|C|ket> before the phase */
#define QSB_SW_XSUM 16u          /* nv=2: sums[2] += Im sum_j <bra|X_j|ket> over the gated qubits */
#define QSB_SW_POST_EXPECT 32u   /* nv=1: sums[0] += <psi|C|psi> after the gates */
#define QSB_SW_POST_DINNER 64u   /* nv=2: sums[0] += Im <bra|C|ket> after the gates */
#define QSB_SW_NO_STORE 128u     /* results are not written back */
#define QSB_SW_EXACT 65536u      /* FMA-free, ascending-order arithmetic */
/* between the two gate passes of a merged / bridge visit (qsb_shard_visit) */
#define QSB_SW_MID_PHASE 512u    /* multiply by exp(i * phase_scale * C) */
#define QSB_SW_MID_DINNER 1024u  /* nv=2: sums[1] += Im <bra|C|ket> */
#define QSB_SW_MID_EXPECT 2048u  /* bridge: sums[0] += <ket|C|ket> (then bra = C * ket) */
#define QSB_SW_XSUM2 4096u       /* nv=2: sums[3] += xsum over the second pass's qubits */

/* One window visit of the sharded window chain (paper_2407_13012_b200/dist.py).
 * mode 0: one gate pass Rx(theta1) on positions [lo1, hi1] (+ pre / post ops);
 * mode 1: merged -- pass 1, the mid ops, pass 2 Rx(theta2) on [lo2, hi2];
 * mode 2: bridge -- pass 1 on the ket only, <C>, bra = C * ket, pass 2 on both.
 * window: 0 = the A window (local bits 0..11), else a B window with its 9 bits at
 * window..window+8.  swap_g > 0 fuses the qubit swap into the store: each output tile
 * (whose top swap_g local bits are c) goes to out0[c] (out1[c] for the bra) at
 * (local & (2^(n-swap_g)-1)) | (swap_rank << (n-swap_g)) -- peer shards' buffers over
 * NVLink (P2P), or chunk c of a local staging buffer for an all-to-all. */
typedef struct qsb_shard_visit {
  int nv, mode, window;
  int lo1, hi1;
  double theta1;
  int lo2, hi2;
  double theta2;
  unsigned flags;
  double phase_scale;
  int swap_g, swap_rank;
  double* out0[8];
  double* out1[8];
} qsb_shard_visit;

typedef struct qsb_ctx qsb_ctx;
typedef struct qsb_table qsb_table;
typedef struct qsb_nccl qsb_nccl; /* an NCCL communicator bound to a context (nccl.cu) */

/* ---------------------------------------------------------------- errors */
const char* qsb_last_error(void);
int qsb_abi_version(void);
/* 1 when the library carries the A/B experiment sweep families (-DQSB_VARIANTS) */
int qsb_has_variants(void);

/* ------------------------------------------------------ device / context */
int qsb_device_count(int* out);
/* one context = one device + one CUDA stream + scratch (backend.py:35 BackendContext) */
int qsb_ctx_create(int device, qsb_ctx** out);
int qsb_ctx_destroy(qsb_ctx* ctx);
int qsb_ctx_sync(qsb_ctx* ctx);
int qsb_ctx_device(qsb_ctx* ctx, int* device);
/* SM count and free/total device memory, for sizing */
int qsb_ctx_info(qsb_ctx* ctx, int* num_sms, uint64_t* free_bytes, uint64_t* total_bytes);
/* device-side timing on the context stream (CUDA events) */
int qsb_timer_start(qsb_ctx* ctx);
int qsb_timer_stop(qsb_ctx* ctx, double* ms);
/* live per-kernel profile: CUDA events around every fused sweep launched between
 * begin and end.  out[3k..3k+2] = {launches, total ms, algorithmic bytes} for
 * kind k (0: single-vector sweep, 1: bra/ket sweep). */
int qsb_prof_begin(qsb_ctx* ctx);
int qsb_prof_end(qsb_ctx* ctx, double* out, int nkinds);
/* host<->device bytes the library has copied on this context (monotone) */
int qsb_ctx_xfer(qsb_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* number of qsb kernel launches issued on this context (monotone) */
int qsb_ctx_launches(qsb_ctx* ctx, uint64_t* out);

/* ----------------------------------------------------- memory (backend.py allocation hooks) */
/* buffers <= 1 GiB come from the device's stream-ordered pool (cudaMallocAsync on the
 * context stream; QSB_NO_MEMPOOL=1: cudaMalloc); qsb_alloc_ipc always uses cudaMalloc
 * (buffers exported with qsb_ipc_handle) */
int qsb_alloc(qsb_ctx* ctx, uint64_t bytes, void** dptr);            /* np.empty, backend.py:133,165 */
int qsb_alloc_ipc(qsb_ctx* ctx, uint64_t bytes, void** dptr);
int qsb_free(qsb_ctx* ctx, void* dptr);                              /* eager release (StateBuffer.free) */
/* Give back to the driver what the library keeps for reuse on `device`: the large-block
 * cache of freed multi-GiB buffers, idle contexts' forward checkpoints and the
 * stream-ordered pool's free memory (no reference counterpart: the reference's arrays
 * are numpy's).  For callers that hand the GPU to another library. */
int qsb_release_cached_memory(int device);
/* CUDA IPC of device buffers for the sharded walk's fused qubit swap (dist.py):
 * export a 64-byte handle, open a peer process's buffer, close it; qsb_device_sync
 * waits for every kernel of this process (peer stores included) to complete. */
int qsb_ipc_handle(qsb_ctx* ctx, const void* dptr, void* handle64);
int qsb_ipc_open(qsb_ctx* ctx, const void* handle64, void** dptr);
int qsb_ipc_close(qsb_ctx* ctx, void* dptr);
int qsb_device_sync(qsb_ctx* ctx);
int qsb_h2d(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int qsb_d2h(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int qsb_d2d(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes); /* clone_state, backend.py:149 */
int qsb_h2d_async(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int qsb_d2h_async(qsb_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int qsb_host_alloc(uint64_t bytes, void** hptr);                     /* pinned host memory */
int qsb_host_free(void* hptr);

/* ------------------------------------------------------- the 14-function kernel set
 * Each mirrors qaoasim/kernels/numba_impl.py (file:line in the comment) with the
 * same arithmetic (FMA-free, same association), so results are bit-identical to
 * the "accelerated" set on identical inputs (phase factors: see qsb_phase_by_table). */
int qsb_fill_plus(qsb_ctx* ctx, double* amps, uint64_t len);                          /* :40-44 */
/* amps *= cos(-gamma*t)+i sin(-gamma*t).  Integer-valued tables with a small range
 * use a host-libm LUT (bit-identical to numba); otherwise device sincos. :47-51 */
int qsb_phase_by_table(qsb_ctx* ctx, double* amps, const double* table, uint64_t len, double gamma);
int qsb_diag_scale(qsb_ctx* ctx, double* amps, const double* table, uint64_t len);    /* :54-57 */
int qsb_rx_qubit(qsb_ctx* ctx, double* amps, uint64_t len, int j, double c, double s); /* :60-72 */
int qsb_weighted_probs(qsb_ctx* ctx, const double* amps, const double* table, double* out, uint64_t len); /* :75-79 */
int qsb_probs(qsb_ctx* ctx, const double* amps, double* out, uint64_t len);           /* :82-86 */
/* neighbour-pair tree with zero padding, bit-identical to tree_sum :114-126 */
int qsb_tree_sum(qsb_ctx* ctx, const double* vals, uint64_t len, double* out);
int qsb_reduce_min(qsb_ctx* ctx, const double* vals, uint64_t len, double* out);      /* :129-136 */
int qsb_reduce_max(qsb_ctx* ctx, const double* vals, uint64_t len, double* out);      /* :138-144 */
int qsb_inner(qsb_ctx* ctx, const double* a, const double* b, uint64_t len, double out[2]);          /* :147-170 */
int qsb_diag_inner(qsb_ctx* ctx, const double* a, const double* table, const double* b, uint64_t len, double out[2]); /* :173-197 */
int qsb_xsum(qsb_ctx* ctx, const double* a, const double* b, uint64_t len, int n_qubits, double out[2]); /* :200-226 */
int qsb_precompute_table(qsb_ctx* ctx, const double* weights, const int64_t* masks, uint64_t num_terms,
                         double* out, uint64_t len);                                   /* :229-238 (host w/m) */
int qsb_pairwise_level(qsb_ctx* ctx, const double* src, double* dst, uint64_t dst_len); /* :241-244 */

/* ------------------------------------------------------- cost table object
 * costpoly.precompute (costpoly.py:126-133): fill the 2^n table on device, record
 * min/max, and — when every value is an integer and max-min < 65536 — a compact
 * uint8/uint16 index table (value = min + idx) used by the fused sweeps for
 * 1-2 B/amp table traffic and exact host-libm phase LUTs. `values` is caller
 * owned (the RealBuffer of CostTable.values). */
int qsb_table_create(qsb_ctx* ctx, int n, const double* weights, const int64_t* masks, uint64_t num_terms,
                     double* values, double* min_out, double* max_out, qsb_table** out);
/* shard of a 2^n_global table for a sharded statevector: local index i of `rank`
 * evaluates x = (i & (2^b-1)) | (rank << s1) | ((i >> b) << s2) */
int qsb_table_create_mapped(qsb_ctx* ctx, int n_global, int n_local, const double* weights, const int64_t* masks,
                            uint64_t num_terms, int b, int s1, int s2, uint64_t rank, double* values,
                            double* min_out, double* max_out, qsb_table** out);
/* wrap an already-filled device table (e.g. uploaded by the user) */
int qsb_table_wrap(qsb_ctx* ctx, int n, double* values, double* min_out, double* max_out, qsb_table** out);
int qsb_table_destroy(qsb_table* t);
/* 0: fp64 + device sincos, 1: uint8 index, 2: uint16 index */
int qsb_table_kind(qsb_table* t, int* kind, int* num_values);
/* phase_by_table through a table object: exact host-libm LUT when compact */
int qsb_table_phase(qsb_ctx* ctx, qsb_table* t, double* amps, double gamma);
/* host-only: the LUT entries (cos, sin)(-gamma * (vmin + k)) the library builds */
int qsb_phase_lut_host(double gamma, double vmin, int nvals, double* out);

/* ------------------------------------------------------- fused hot path
 * Layer = phase exp(-i gamma C) then Rx(-2 beta) on every qubit (circuit.py:98-103).
 * The phase is fused into the first mixer sweep; ~12 qubits are applied per HBM
 * sweep (shared-memory exchange between register-resident butterfly phases). */
int qsb_simulate(qsb_ctx* ctx, qsb_table* t, double* amps, int p, const double* gammas,
                 const double* betas, unsigned flags);
/* simulate + <psi|C|psi> taken from the last sweep (circuit.expectation, circuit.py:116-118) */
int qsb_simulate_expect(qsb_ctx* ctx, qsb_table* t, double* amps, int p, const double* gammas,
                        const double* betas, unsigned flags, double* expect_out);
/* Rx(theta) on every qubit of amps (backend.apply_rx_layer, backend.py:200-207) */
int qsb_rx_layer(qsb_ctx* ctx, double* amps, int n, double theta, unsigned flags);
/* Rx(theta) on qubits [lo, hi] with fused ops (QSB_SW_*); sums[3] = partial sums
 * (see fused.cu).  Building block of the sharded walk. */
int qsb_layer_sweeps(qsb_ctx* ctx, qsb_table* t, double* v0, double* v1, int nv, int n, int n_global, int lo,
                     int hi, double theta, unsigned flags, double phase_scale, double* sums);
/* One visit of the sharded window chain (fast mode); sums[4] = {<C> or post / mid
 * <bra|C|ket>... see qsb_shard_visit: slot 0 <C> / post dinner / bridge <C>, 1 pre or mid
 * Im<bra|C|ket>, 2 xsum of pass 1, 3 xsum of pass 2}.  n = local qubits of the shard. */
int qsb_shard_visit_run(qsb_ctx* ctx, qsb_table* t, double* v0, double* v1, int n, int n_global,
                        const qsb_shard_visit* d, double* sums);
/* Many small registers (n <= 11 each) in ONE launch, one CTA per instance (the
 * paper's many-graphs regime; no reference counterpart -- the reference runs handles
 * one by one, cli.py bench --jobs).  Instance k: table tables[k], state kets[k]
 * (written with the final ket), depth ps[k], angles gammas/betas concatenated in
 * instance order.  mode 0 simulate, 1 + <C>, 2 + gradient.  out (host): per instance
 * 1 + 2p doubles: <C> (unclamped), d_gamma[p], d_beta[p]. */
int qsb_small_batch(qsb_ctx* ctx, int count, qsb_table* const* tables, double* const* kets, const int* ps,
                    const double* gammas, const double* betas, int mode, double* out);
/* Many mid-size registers (12 <= n, each on its own context) -- the paper's
 * many-graphs regime above the one-CTA size (cli.py bench --jobs runs handles one per
 * thread).  Instance k: context ctxs[k] (its own CUDA stream), table tables[k], ket /
 * bra kets[k] / bras[k], depth ps[k], angles concatenated in instance order.  Every
 * instance's window chain (as qsb_value_and_grad) is issued before any is awaited, so
 * instances whose sweeps fill only a few SMs (2^(n-12) tiles) run concurrently.
 * out (host): per instance 1 + 2p doubles: <C> (unclamped), d_gamma[p], d_beta[p]. */
int qsb_value_and_grad_many(int count, qsb_ctx* const* ctxs, qsb_table* const* tables, double* const* kets,
                            double* const* bras, const int* ps, const double* gammas, const double* betas,
                            double* out);
/* <psi|C|psi> (circuit.expectation_of_state, circuit.py:106-113, without the clamp) */
int qsb_expectation(qsb_ctx* ctx, qsb_table* t, const double* amps, unsigned flags, double* out);
/* expectation + adjoint gradient (adjoint.py:37-77): one forward, one backward walk
 * over exactly two statevectors (ket = amps, bra = caller-provided scratch).
 * If `skip_forward` != 0 the caller guarantees amps already holds simulate(params).
 * value may be NULL.  d_gammas/d_betas: host arrays of length p. */
int qsb_value_and_grad(qsb_ctx* ctx, qsb_table* t, double* ket, double* bra, int p,
                       const double* gammas, const double* betas, unsigned flags, int skip_forward,
                       double* value, double* d_gammas, double* d_betas);
/* sampling (backend.sample_indices, backend.py:261-299 + sampling.draw): probability
 * tree with the reference's pairwise association, splitmix64 uniforms (rng.py:30-37),
 * root-to-leaf descent; costs gathered from the table on device.
 * t may be NULL (indices only; cost_out ignored).
 * Writes total (tree root) before checking normalisation; returns QSB_EINVAL with
 * "not normalized" when |root-1| > 1e-9.  idx/cost are HOST arrays of `shots`. */
int qsb_sample(qsb_ctx* ctx, qsb_table* t, const double* amps, int n, uint64_t shots, uint64_t seed,
               int64_t* idx_out, double* cost_out, double* total_out);

/* qsb_sample for a flip-symmetric state held as its lower half (the Z2 reduction:
 * psi(x) = psi(~x), half_amps = psi(x) for x < 2^(n-1); same role as qsb_sample,
 * backend.py:261-299).  The upper half of the reference's tree mirrors the lower half
 * node for node, so only the lower half's levels are built; indices, costs and the
 * root are bit-identical to qsb_sample on the materialised state. */
int qsb_sample_sym(qsb_ctx* ctx, qsb_table* t, const double* half_amps, int n, uint64_t shots, uint64_t seed,
                   int64_t* idx_out, double* cost_out, double* total_out);

/* Sharded sampling (no reference counterpart: the reference samples one host array,
 * backend.py:261-299; SURVEY.md §8(e) "Sampling across GPUs").  A shard builds the
 * levels of its 2^n_local-amplitude subtree (kept in the context) and reports its
 * root; the caller combines the shard roots with the reference's pairwise
 * association, draws u = U(seed, s) * total, descends the levels above the shards and
 * hands each shard the residual u of the shots that land in it. */
int qsb_sample_tree(qsb_ctx* ctx, const double* amps, int n_local, double* root_out);
/* Descend the tree built by qsb_sample_tree for `count` shots with residuals u[]
 * (HOST array); local indices and (t != NULL) costs go to HOST arrays. */
int qsb_sample_descend(qsb_ctx* ctx, qsb_table* t, const double* amps, int n_local, uint64_t count, const double* u,
                       int64_t* idx_out, double* cost_out);

/* Standalone qubit swap of a sharded statevector (SURVEY.md §8(e) "The collective";
 * no reference counterpart -- the reference is single-array): chunk c
 * (chunk_amps amplitudes at src + c * chunk_amps) goes to dsts[c] + dst_off_amps, for
 * c < nchunks <= 8, in one kernel.  dsts may be CUDA-IPC-mapped peer buffers (the
 * stores cross NVLink; complete with qsb_device_sync + a host barrier). */
int qsb_scatter_chunks(qsb_ctx* ctx, const double* src, uint64_t chunk_amps, int nchunks, void* const* dsts,
                       uint64_t dst_off_amps);
/* Native NCCL transport of the same swap (no reference counterpart; SURVEY.md §8(e)
 * "The collective", the non-P2P mode of dist.py TorchExchanger).  libnccl.so.2 is
 * opened at run time; without it these return QSB_EINVAL with the reason.
 * unique_id: 128 bytes (rank 0 creates it, the caller broadcasts it); init binds the
 * communicator to ctx's device and stream; all_to_all: dst chunk c <- rank c's src
 * chunk `rank` (chunk_amps complex128 amplitudes per chunk, nranks chunks), one NCCL
 * group of send/recv pairs on the context stream (stream-ordered, no host sync). */
int qsb_nccl_version(int* version);
int qsb_nccl_unique_id(void* id);
int qsb_nccl_init(qsb_ctx* ctx, const void* id, int nranks, int rank, qsb_nccl** out);
int qsb_nccl_all_to_all(qsb_nccl* c, const double* src, double* dst, uint64_t chunk_amps);
/* Wait for the context stream's swaps, polling ncclCommGetAsyncError; on an NCCL error or
 * after timeout_ms (< 0: none) the communicator is aborted (ncclCommAbort) and an error
 * returned instead of a hang (failure detection). */
int qsb_nccl_wait(qsb_nccl* c, int64_t timeout_ms);
int qsb_nccl_destroy(qsb_nccl* c);
/* amps[i] = re + i*im (a shard's part of |+> is 1/sqrt(2^n_global), fill_plus
 * numba_impl.py:40-44 for the whole register) */
int qsb_fill_const(qsb_ctx* ctx, double* amps, uint64_t len, double re, double im);
/* Drop the table's fp64 values (kind 1/2 only): every later use reads the compact
 * index (T = vmin + idx, exact for integral tables).  Lets a sharded handle free the
 * 8 B/amp fp64 copy of each layout's table (the caller frees the memory). */
int qsb_table_detach_values(qsb_table* t);
/* Z2 reduction (flip-symmetric cost tables, C(x) = C(~x): every MaxCut).  The state
 * then keeps psi(x) = psi(~x), and the fused paths evolve only x < 2^(n-1).
 * qsb_table_symmetric: 1 when the table is flip-symmetric bit for bit.
 * qsb_state_mirror: write the upper half from the lower, psi(2^(n-1)+y) = psi(2^(n-1)-1-y).
 * qsb_ctx_last_half: 1 when the context's last simulate left the upper half unwritten. */
int qsb_table_symmetric(qsb_table* t, int* sym);
int qsb_state_mirror(qsb_ctx* ctx, double* amps, int n);
int qsb_ctx_last_half(qsb_ctx* ctx, int* half);

#ifdef __cplusplus
}
#endif
#endif /* QSB_H */
