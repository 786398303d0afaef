"""Sharded statevectors across G = 2^g GPUs (future work in the
reference, PAPER.md:234 / SPEC.md:155).

Shard r of an n-qubit state holds N_l = 2^(n-g) amplitudes.  Two layouts alternate:

  layout A: local index i <-> global x = i | (r << n_l)
  layout B: the top g local bits and the rank bits trade places:
            x = (i & (2^(n_l-g)-1)) | (r << (n_l-g)) | ((i >> (n_l-g)) << n_l)

Going A <-> B is one all-to-all of equal contiguous chunks (chunk c of shard r, i.e.
the amplitudes whose top g local bits are c, goes to shard c and lands as its chunk
r) — `torch.distributed.all_to_all_single` over NCCL/NVLink with one shard per
process, or device copies when several virtual shards share one GPU (tests).

Every layer's mixer is Rx(theta) on *every* qubit, so which qubit sits at which
position does not matter for the gates: a layer applies the phase (table of the
current layout) and Rx to all n_l local positions, swaps, then applies Rx to the g
positions that just arrived.  The next layer starts in the other layout.  The
adjoint walk does the same with the bra/ket pair; the fused contractions
(<C>, <bra|C|ket>, sum_j <bra|X_j|ket>) are per-shard partial sums combined in rank
order.  `program()` is that schedule as data, executed on the GPU by `_run` and
emulated in numpy by the tests (tests/test_dist_host.py).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib, backend, circuit, costpoly, rng, sampling
from ._lib import DeviceArray, call
from .errors import ContractViolation
from .kernels import b200

# fused-op flags of qsb_layer_sweeps (include/qsb.h)
PLUS, PRE_PHASE, BRA_FROM_KET, PRE_DINNER, XSUM, POST_EXPECT, POST_DINNER, NO_STORE = (
    1, 2, 4, 8, 16, 32, 64, 128)
EXACT = 65536


# ---------------------------------------------------------------- layouts
def index_map(layout: int, n: int, g: int, rank: int) -> tuple[int, int, int, int]:
    """(b, s1, s2, rank) such that x = (i & (2^b-1)) | (rank << s1) | ((i >> b) << s2)."""
    n_l = n - g
    if layout == 0:
        return n_l, n_l, 0, rank
    return n_l - g, n_l - g, n_l, rank


def global_index(layout: int, n: int, g: int, rank: int, i: np.ndarray) -> np.ndarray:
    b, s1, s2, r = index_map(layout, n, g, rank)
    i = np.asarray(i, dtype=np.int64)
    return (i & ((1 << b) - 1)) | (r << s1) | ((i >> b) << s2)


# ---------------------------------------------------------------- the schedule
@dataclass(frozen=True)
class Sweeps:
    nv: int            # 1: ket only, 2: bra and ket
    lo: int            # gated local positions [lo, hi]
    hi: int
    theta: float       # Rx(theta)
    flags: int
    phase: float       # exp(i * phase * C) before the gates when PRE_PHASE
    layer: int         # QAOA layer index (0-based)
    tag: str           # "fwd" / "fwd_tail" / "bwd" / "bwd_tail"


@dataclass(frozen=True)
class Swap:
    nv: int


def program(n: int, g: int, gammas, betas, want_value: bool, want_grad: bool):
    """The sharded forward (+ adjoint) walk as a list of Sweeps / Swap steps."""
    n_l = n - g
    p = len(gammas)
    steps: list = []
    for i in range(p):
        f = PRE_PHASE | (PLUS if i == 0 else 0)
        steps.append(Sweeps(1, 0, n_l - 1, -2.0 * betas[i], f, -gammas[i], i, "fwd"))
        steps.append(Swap(1))
        tail = POST_EXPECT if (i == p - 1 and want_value) else 0
        steps.append(Sweeps(1, n_l - g, n_l - 1, -2.0 * betas[i], tail, 0.0, i, "fwd_tail"))
    if not want_grad:
        return steps
    for i in range(p - 1, -1, -1):
        f = XSUM | (BRA_FROM_KET if i == p - 1 else PRE_DINNER | PRE_PHASE)
        ph = gammas[i + 1] if i < p - 1 else 0.0
        steps.append(Sweeps(2, 0, n_l - 1, 2.0 * betas[i], f, ph, i, "bwd"))
        steps.append(Swap(2))
        tail = XSUM | ((POST_DINNER | NO_STORE) if i == 0 else 0)
        steps.append(Sweeps(2, n_l - g, n_l - 1, 2.0 * betas[i], tail, 0.0, i, "bwd_tail"))
    return steps


def collect(steps, sums_per_step, p: int):
    """Fold per-step contraction sums (already combined over shards) into
    (value, d_gammas, d_betas) exactly as the single-GPU walk defines them."""
    value = None
    dg = np.zeros(p)
    db = np.zeros(p)
    xs = np.zeros(p)
    for st, s in zip(steps, sums_per_step):
        if not isinstance(st, Sweeps):
            continue
        if st.nv == 1 and (st.flags & POST_EXPECT):
            value = s[0]
        if st.nv == 2:
            xs[st.layer] += s[2]
            if st.flags & PRE_DINNER:
                dg[st.layer + 1] = 2.0 * s[1]
            if st.flags & POST_DINNER:
                dg[st.layer] = 2.0 * s[0]
    db[:] = -2.0 * xs
    return value, dg, db


# ---------------------------------------------------------------- the window chain (fast mode)
MID_PHASE, MID_DINNER, MID_EXPECT, XSUM2 = 512, 1024, 2048, 4096
PLAIN, MERGED, BRIDGE = 0, 1, 2


@dataclass(frozen=True)
class Visit:
    """One window visit on every shard (qsb_shard_visit, include/qsb.h)."""

    nv: int
    mode: int          # PLAIN / MERGED / BRIDGE
    window: int        # 0: A window (bits 0..11), else a B window's first bit
    lo1: int
    hi1: int
    theta1: float
    lo2: int
    hi2: int
    theta2: float
    flags: int
    phase: float
    swap: bool         # the qubit swap (layout A <-> B) follows this visit
    routes: tuple      # (slot, kind, layer): kind 0 <C>, 1 d_gamma (x2), 2 d_beta (x-2)


def shard_windows(n_l: int) -> list[tuple[int, int, int]]:
    """Visit order of one layer's windows as (window, lo, hi): the top B window first
    (it also takes the previous layer's g swapped-in qubits), the A window last (its
    tiles hold fixed top bits, so the swap can follow -- or be fused into -- it)."""
    if n_l < 21:
        raise ContractViolation(f"the sharded chain needs >= 21 local qubits (n_l={n_l})")
    wins = [(0, 0, 11)]
    s = 12
    while s <= n_l - 1:
        glo = min(s, n_l - 9)
        wins.append((glo, glo, glo + 8))
        s += 9
    order = list(reversed(wins))
    out, covered = [], set()
    for w, lo, hi in order:
        pos = [q for q in range(lo, hi + 1) if q not in covered]
        covered.update(pos)
        if pos:
            out.append((w, pos[0], pos[-1]))
    return out


def chain_program(n: int, g: int, gammas, betas, want_value: bool, want_grad: bool) -> list[Visit]:
    """The sharded walk as window visits.  A layer gates its local positions window by
    window (top B window, middle B windows, A window), then the top g local bits and
    the rank bits trade places (one all-to-all, or fused into the A visit's store), and
    the g qubits that arrived are gated in the next visit of the top window -- merged
    with the next layer (phase between the passes), the bridge to the backward walk, or
    a final tail.  Per layer: K visits + 1 swap (the per-position schedule of program()
    needs K + 1 sweeps + 1 swap)."""
    n_l = n - g
    p = len(gammas)
    wins = shard_windows(n_l)
    top_w, top_lo, top_hi = wins[0]
    arr_lo, arr_hi = n_l - g, n_l - 1
    V = []
    for i in range(p):
        th = -2.0 * betas[i]
        for k, (w, lo, hi) in enumerate(wins):
            last = k == len(wins) - 1
            if k == 0 and i == 0:
                V.append(Visit(1, PLAIN, w, lo, hi, th, 0, 0, 0.0, PLUS | PRE_PHASE, -gammas[0], False, ()))
            elif k == 0:
                V.append(Visit(1, MERGED, w, arr_lo, arr_hi, -2.0 * betas[i - 1], lo, hi, th, MID_PHASE, -gammas[i],
                               False, ()))
            else:
                V.append(Visit(1, PLAIN, w, lo, hi, th, 0, 0, 0.0, 0, 0.0, last, ()))
    if not want_grad:
        V.append(Visit(1, PLAIN, top_w, arr_lo, arr_hi, -2.0 * betas[p - 1], 0, 0, 0.0,
                       POST_EXPECT if want_value else 0, 0.0, False, ((0, 0, 0),) if want_value else ()))
        return V
    for i in range(p - 1, -1, -1):
        th = 2.0 * betas[i]
        for k, (w, lo, hi) in enumerate(wins):
            last = k == len(wins) - 1
            if k == 0 and i == p - 1:
                routes = ((3, 2, i),) + (((0, 0, 0),) if want_value else ())
                V.append(Visit(2, BRIDGE, w, arr_lo, arr_hi, -2.0 * betas[p - 1], lo, hi, th,
                               XSUM2 | (MID_EXPECT if want_value else 0), 0.0, False, routes))
            elif k == 0:
                V.append(Visit(2, MERGED, w, arr_lo, arr_hi, 2.0 * betas[i + 1], lo, hi, th,
                               XSUM | MID_DINNER | MID_PHASE | XSUM2, gammas[i + 1], False,
                               ((2, 2, i + 1), (1, 1, i + 1), (3, 2, i))))
            else:
                V.append(Visit(2, PLAIN, w, lo, hi, th, 0, 0, 0.0, XSUM, 0.0, last, ((2, 2, i),)))
    V.append(Visit(2, PLAIN, top_w, arr_lo, arr_hi, 2.0 * betas[0], 0, 0, 0.0, XSUM | POST_DINNER | NO_STORE, 0.0,
                   False, ((2, 2, 0), (0, 1, 0))))
    return V


def collect_chain(visits, sums, p: int):
    value = None
    dg = np.zeros(p)
    db = np.zeros(p)
    for v, s in zip(visits, sums):
        for slot, kind, layer in v.routes:
            if kind == 0:
                value = s[slot]
            elif kind == 1:
                dg[layer] += 2.0 * s[slot]
            else:
                db[layer] += -2.0 * s[slot]
    return value, dg, db


class _ShardVisit(C.Structure):
    _fields_ = [("nv", C.c_int), ("mode", C.c_int), ("window", C.c_int), ("lo1", C.c_int), ("hi1", C.c_int),
                ("theta1", C.c_double), ("lo2", C.c_int), ("hi2", C.c_int), ("theta2", C.c_double),
                ("flags", C.c_uint), ("phase_scale", C.c_double), ("swap_g", C.c_int), ("swap_rank", C.c_int),
                ("out0", C.c_void_p * 8), ("out1", C.c_void_p * 8)]


# ---------------------------------------------------------------- exchangers
def _ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * len(ptrs))()
    for i, p_ in enumerate(ptrs):
        arr[i] = p_
    return arr


class VirtualExchanger:
    """All G shards live in this process on one device: the all-to-all is one chunk
    scatter kernel per shard (qsb_scatter_chunks) into the other shards' spares."""

    fused = True  # the swap is fused into the A visit's stores (shard buffers are plain device memory)

    def __init__(self, g: int):
        self.G = 1 << g
        self.ranks = list(range(self.G))

    def setup(self, handle) -> None:
        pass

    def _setup_nccl(self, handle, force: bool = False) -> None:
        """libqsb's own NCCL communicator for the all-to-all swaps: rank 0's unique id is
        broadcast, every rank initialises, and all agree (one all_reduce) -- any failure
        leaves every rank on torch.distributed's all_to_all_single."""
        import os

        import torch

        mode = os.environ.get("QSB_SHARD_NCCL", "native")  # native | torch | force (also over gloo: tests)
        force = force or mode == "force"
        if (self.cpu and not force) or mode == "torch":
            return
        self._ctx = handle.ctx.device.handle
        uid = np.zeros(129, dtype=np.uint8)
        if self.rank == 0:
            try:
                call("qsb_nccl_unique_id", uid.ctypes.data)
                uid[128] = 1
            except Exception:  # noqa: BLE001 -- decided collectively below
                uid[128] = 0
        t = torch.as_tensor(uid, device=self._tdev())
        self.dist.broadcast(t, src=0)
        uid = np.ascontiguousarray(t.cpu().numpy())
        comm = C.c_void_p()
        ok = int(uid[128] == 1)
        if ok:
            try:
                call("qsb_nccl_init", self._ctx, uid.ctypes.data, self.G, self.rank, C.byref(comm))
            except Exception:  # noqa: BLE001
                ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self._tdev())
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            self._nccl = comm.value
        elif comm.value:
            call("qsb_nccl_destroy", comm.value)

    def targets(self, name: str, spare: list[DeviceArray]) -> list[int]:
        """where the fused swap store sends tile chunk c: shard c's spare buffer"""
        return [b.ptr for b in spare]

    def commit(self, name: str, live: list[DeviceArray], spare: list[DeviceArray]) -> None:
        for k in range(len(live)):  # the spare buffers now hold the swapped state
            live[k].ptr, spare[k].ptr = spare[k].ptr, live[k].ptr

    def combine(self, per_rank_sums: list[np.ndarray]) -> np.ndarray:
        total = np.zeros_like(per_rank_sums[0])
        for s in per_rank_sums:  # rank order: deterministic
            total = total + s
        return total

    def gather(self, local: list[float]) -> list[float]:
        """one value per rank, rank order (all ranks are local)"""
        return list(local)

    def owned_sum(self, *arrays: np.ndarray) -> tuple[np.ndarray, ...]:
        """element-wise sum over ranks of arrays each rank filled only where it owns the entry"""
        return arrays

    def all_max(self, *vals: float) -> tuple[float, ...]:
        return vals

    def swap_vec(self, name: str, live: list[DeviceArray], spare: list[DeviceArray]) -> None:
        """standalone qubit swap of one vector: shard r's chunk c -> shard c's chunk r"""
        G = self.G
        chunk = len(live[0]) // G
        dsts = _ptr_array([b.ptr for b in spare])
        for r in range(G):
            call("qsb_scatter_chunks", live[r].dctx.handle, live[r].ptr, chunk, G, dsts, r * chunk)
        self.commit(name, live, spare)


class TorchExchanger:
    """One shard per process (torchrun).  The qubit swap is fused into the A visit's
    stores when p2p=True / QSB_SHARD_P2P=1: every process opens its peers' spare buffers
    through CUDA IPC and the sweep kernel writes each output tile straight into the shard
    that owns it after the swap (NVLink P2P stores overlapped with the sweep; no separate
    pass).  Swaps outside a fused visit (a draw after an odd number of layers, exact
    mode, shards below 21 local qubits) then run qsb_scatter_chunks into the same peer
    buffers.  Without P2P the swap is an all-to-all after the A visit: libqsb's own NCCL
    communicator (qsb_nccl_*, one group of send/recv pairs on the context stream, no host
    sync) when libnccl loads, else torch.distributed's all_to_all_single
    (QSB_SHARD_NCCL=torch forces it); with a gloo process group (tests: two processes on
    one GPU) the host-side collectives run on CPU tensors and the non-P2P swap is staged
    through host memory."""

    def __init__(self, g: int, dist, device: int, p2p: bool | None = None):
        import os

        self.G = 1 << g
        self.dist = dist
        self.rank = dist.get_rank()
        self.ranks = [self.rank]
        self.device = device
        if dist.get_world_size() != self.G:
            raise ContractViolation(f"world size {dist.get_world_size()} != 2^g = {self.G}")
        if p2p is None:
            p2p = os.environ.get("QSB_SHARD_P2P", "0") == "1"
        self.fused = bool(p2p)
        self.cpu = dist.get_backend() == "gloo"
        self._peers: dict[str, list[list[int]]] = {}
        self._parity: dict[str, int] = {}
        self._opened: list[int] = []
        self._ctx = None
        self._nccl = None  # qsb_nccl communicator (non-P2P swaps over NCCL)

    def _tdev(self) -> str:
        return "cpu" if self.cpu else f"cuda:{self.device}"

    def setup(self, handle) -> None:
        """P2P mode: export this shard's live/spare buffers, open every peer's.  If any
        rank cannot (no peer access), every rank falls back to the all-to-all.

        Every rank runs the same collectives whatever fails locally: the handles are
        exported first (a failure only clears this rank's ok byte), exchanged in ONE
        all_gather, opened with no collective in between, and the outcome agreed by
        one all_reduce."""
        if not self.fused:
            self._setup_nccl(handle)
            return
        import torch

        self._ctx = handle.ctx.device.handle
        bufs = (("ket", handle.ket[0], handle.scratch[0]), ("bra", handle.bra[0], handle.scratch_bra[0]))
        mine = np.zeros(257, dtype=np.uint8)
        try:
            for i, (_, b0, b1) in enumerate(bufs):
                call("qsb_ipc_handle", self._ctx, b0.ptr, mine[128 * i:128 * i + 64].ctypes.data)
                call("qsb_ipc_handle", self._ctx, b1.ptr, mine[128 * i + 64:128 * i + 128].ctypes.data)
            mine[256] = 1
        except Exception:  # noqa: BLE001 -- decided collectively below
            mine[256] = 0
        t = torch.as_tensor(mine, device=self._tdev())
        out = [torch.empty_like(t) for _ in range(self.G)]
        self.dist.all_gather(out, t)
        handles = [np.ascontiguousarray(o.cpu().numpy()) for o in out]
        ok = int(all(h[256] == 1 for h in handles))
        if ok:
            try:
                for i, (name, b0, b1) in enumerate(bufs):
                    ptrs = []
                    for r in range(self.G):
                        if r == self.rank:
                            ptrs.append([b0.ptr, b1.ptr])
                            continue
                        pp = []
                        for off in (128 * i, 128 * i + 64):
                            p_ = C.c_void_p()
                            call("qsb_ipc_open", self._ctx, handles[r][off:off + 64].ctypes.data, C.byref(p_))
                            pp.append(p_.value)
                            self._opened.append(p_.value)
                        ptrs.append(pp)
                    self._peers[name] = ptrs
                    self._parity[name] = 0
            except Exception:  # noqa: BLE001
                ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self._tdev())
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            self.close()
            self._peers, self._parity = {}, {}
            self.fused = False
            self._setup_nccl(handle)

    def _setup_nccl(self, handle, force: bool = False) -> None:
        """libqsb's own NCCL communicator for the all-to-all swaps: rank 0's unique id is
        broadcast, every rank initialises, and all agree (one all_reduce) -- any failure
        leaves every rank on torch.distributed's all_to_all_single."""
        import os

        import torch

        mode = os.environ.get("QSB_SHARD_NCCL", "native")  # native | torch | force (also over gloo: tests)
        force = force or mode == "force"
        if (self.cpu and not force) or mode == "torch":
            return
        self._ctx = handle.ctx.device.handle
        uid = np.zeros(129, dtype=np.uint8)
        if self.rank == 0:
            try:
                call("qsb_nccl_unique_id", uid.ctypes.data)
                uid[128] = 1
            except Exception:  # noqa: BLE001 -- decided collectively below
                uid[128] = 0
        t = torch.as_tensor(uid, device=self._tdev())
        self.dist.broadcast(t, src=0)
        uid = np.ascontiguousarray(t.cpu().numpy())
        comm = C.c_void_p()
        ok = int(uid[128] == 1)
        if ok:
            try:
                call("qsb_nccl_init", self._ctx, uid.ctypes.data, self.G, self.rank, C.byref(comm))
            except Exception:  # noqa: BLE001
                ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self._tdev())
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            self._nccl = comm.value
        elif comm.value:
            call("qsb_nccl_destroy", comm.value)

    def targets(self, name: str, spare: list[DeviceArray]) -> list[int]:
        par = self._parity[name]
        return [self._peers[name][c][1 - par] for c in range(self.G)]

    def commit(self, name: str, live: list[DeviceArray], spare: list[DeviceArray]) -> None:
        call("qsb_device_sync", self._ctx)  # our stores into the peers are complete
        self.dist.barrier()                  # ... and everybody's into ours
        self._parity[name] ^= 1
        live[0].ptr, spare[0].ptr = spare[0].ptr, live[0].ptr

    def close(self) -> None:
        if self._nccl:
            try:
                call("qsb_nccl_destroy", self._nccl)
            except Exception:  # noqa: BLE001 -- best effort at teardown
                pass
            self._nccl = None
        for p_ in self._opened:
            try:
                call("qsb_ipc_close", self._ctx, p_)
            except Exception:  # noqa: BLE001 -- best effort at teardown
                pass
        self._opened = []

    def combine(self, per_rank_sums: list[np.ndarray]) -> np.ndarray:
        import torch

        mine = torch.tensor(per_rank_sums[0], dtype=torch.float64, device=self._tdev())
        out = [torch.empty_like(mine) for _ in range(self.G)]
        self.dist.all_gather(out, mine)
        total = np.zeros_like(per_rank_sums[0])
        for t in out:  # rank order: deterministic, identical on every rank
            total = total + t.cpu().numpy()
        return total

    def gather(self, local: list[float]) -> list[float]:
        import torch

        mine = torch.tensor(local, dtype=torch.float64, device=self._tdev())
        out = [torch.empty_like(mine) for _ in range(self.G)]
        self.dist.all_gather(out, mine)
        return [float(x) for t in out for x in t.cpu().tolist()]

    def owned_sum(self, *arrays: np.ndarray) -> tuple[np.ndarray, ...]:
        import torch

        res = []
        for a in arrays:  # exactly one rank contributes each entry: the sum is exact
            t = torch.as_tensor(a, device=self._tdev())
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
            res.append(t.cpu().numpy())
        return tuple(res)

    def all_max(self, *vals: float) -> tuple[float, ...]:
        import torch

        t = torch.tensor(list(vals), dtype=torch.float64, device=self._tdev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return tuple(float(x) for x in t.tolist())

    def swap_vec(self, name: str, live: list[DeviceArray], spare: list[DeviceArray]) -> None:
        """Standalone qubit swap of one vector (see the class doc): P2P chunk scatter into
        the peers' spare buffers, else an all-to-all (NCCL; host-staged over gloo)."""
        import torch

        v, s = live[0], spare[0]
        chunk = len(v) // self.G
        if self.fused:
            call("qsb_scatter_chunks", self._ctx, v.ptr, chunk, self.G, _ptr_array(self.targets(name, spare)),
                 self.rank * chunk)
            self.commit(name, live, spare)
            return
        if self._nccl:  # stream-ordered on the context stream
            call("qsb_nccl_all_to_all", self._nccl, v.ptr, s.ptr, chunk)
            # failure detection: an NCCL error or a peer that never arrives aborts the
            # communicator and raises here instead of hanging the next host sync
            call("qsb_nccl_wait", self._nccl, int(os.environ.get("QSB_NCCL_TIMEOUT_MS", "600000")))
        elif self.cpu:  # gloo stand-in: D2H, all-to-all of host tensors, H2D into the spare
            host = torch.from_numpy(v.to_host().view(np.float64)).view(self.G, -1)
            recv = torch.empty_like(host)
            self.dist.all_to_all_single(recv, host)
            s.from_host(recv.numpy().reshape(-1).view(np.complex128))
        else:
            v.dctx.sync()  # our stream -> NCCL's stream
            src = torch.as_tensor(_CudaView(v), device=f"cuda:{self.device}").view(self.G, -1)
            dst = torch.as_tensor(_CudaView(s), device=f"cuda:{self.device}").view(self.G, -1)
            self.dist.all_to_all_single(dst, src)
            torch.cuda.synchronize(self.device)
        v.ptr, s.ptr = s.ptr, v.ptr


class _CudaView:
    """__cuda_array_interface__ view of a DeviceArray as float64 pairs (no copy)."""

    def __init__(self, d: DeviceArray):
        self.__cuda_array_interface__ = {
            "shape": (2 * d.length,) if d.dtype == np.complex128 else (d.length,),
            "typestr": "<f8",
            "data": (d.ptr, False),
            "version": 3,
            "strides": None,
            "stream": None,
        }


# ---------------------------------------------------------------- sharded handle
class ShardedHandle:
    """A polynomial's statevector split over 2^g shards (this process holds
    `exchanger.ranks`), with cost tables for both layouts.

    Per-GPU memory (N_l = 2^(n-g) amplitudes per shard): ket, bra and one spare per
    vector for the qubit swap (4 x 16 N_l B) plus each layout's table -- the 1-2 B/amp
    compact index when the table is integral with < 65536 distinct values (the fp64
    copy is built, compacted and freed one layout at a time), else fp64 (8 B/amp).
    n = 34 on 8 GPUs (N_l = 2^31, MaxCut u8 index): 128 GiB + 2 x 2 GiB + the
    sampler's 1 GiB level scratch, ~134 GiB of the B200's ~178 GiB (DESIGN.md (e))."""

    def __init__(self, poly: costpoly.Polynomial, g: int, exchanger, device: int | None = None):
        n = poly.n
        if g < 1:
            raise ContractViolation("sharding needs g >= 1 (use create_handle for one GPU)")
        if g > 3:
            raise ContractViolation(f"at most 8 shards (g <= 3), got g={g}")
        if n - g < 12:
            raise ContractViolation(f"shards need >= 12 local qubits (n={n}, g={g})")
        self.n, self.g, self.n_l = n, g, n - g
        self.poly = poly
        self.ex = exchanger
        self.ctx = backend.create_context("b200", device)
        dctx = self.ctx.device
        N_l = 1 << self.n_l
        self.ranks = list(exchanger.ranks)
        # tables first (their fp64 build buffers are transient), then the statevectors
        w = np.ascontiguousarray(poly.weights, dtype=np.float64)
        m = np.ascontiguousarray(poly.masks, dtype=np.int64)
        self.tables = [[None] * len(self.ranks), [None] * len(self.ranks)]
        lo, hi = np.inf, -np.inf
        self.table_bytes = 0
        for layout in (0, 1):
            for k, r in enumerate(self.ranks):
                vals = DeviceArray(dctx, N_l, np.float64)
                b, s1, s2, rank = index_map(layout, n, g, r)
                mn, mx, ptr = C.c_double(), C.c_double(), C.c_void_p()
                call("qsb_table_create_mapped", dctx.handle, n, self.n_l, w.ctypes.data, m.ctypes.data, w.shape[0],
                     b, s1, s2, rank, vals.ptr, C.byref(mn), C.byref(mx), C.byref(ptr))
                b200._attach(vals, ptr)
                if vals.table.kind != 0:  # the sweeps and the sampler read the compact index only
                    call("qsb_table_detach_values", vals.table.ptr)
                    vals.free()
                    self.table_bytes += N_l * vals.table.kind
                else:
                    self.table_bytes += 8 * N_l
                self.tables[layout][k] = vals
                lo, hi = min(lo, mn.value), max(hi, mx.value)
        self.min_value, self.max_value = self._minmax(lo, hi)
        # statevector buffers: plain cudaMalloc memory (exportable to peer processes)
        self.ket = [DeviceArray(dctx, N_l, np.complex128, ipc=True) for _ in self.ranks]
        self.bra = [DeviceArray(dctx, N_l, np.complex128, ipc=True) for _ in self.ranks]
        self.scratch = [DeviceArray(dctx, N_l, np.complex128, ipc=True) for _ in self.ranks]
        # a fused swap of a bra/ket visit needs a second spare (up front for P2P, whose
        # buffers are exported once; lazily for virtual shards)
        self.scratch_bra = None
        if exchanger.fused and not isinstance(exchanger, VirtualExchanger):
            self.scratch_bra = [DeviceArray(dctx, N_l, np.complex128, ipc=True) for _ in self.ranks]
        self.layout = 0
        self._plus_pending = False  # the ket is |+> by contract but not written (after a gradient)
        exchanger.setup(self)

    def _minmax(self, lo: float, hi: float) -> tuple[float, float]:
        neg_lo, hi = self.ex.all_max(-lo, hi)
        return -neg_lo, hi

    def _spare(self, name: str) -> list[DeviceArray]:
        if name == "ket":
            return self.scratch
        if self.scratch_bra is not None and not isinstance(self.ex, VirtualExchanger):
            return self.scratch_bra  # P2P: the exported bra spares
        return self.scratch

    def _swap(self, nv: int) -> None:
        """standalone qubit swap (layout A <-> B) of the ket (and the bra)"""
        self.ex.swap_vec("ket", self.ket, self._spare("ket"))
        if nv == 2:
            self.ex.swap_vec("bra", self.bra, self._spare("bra"))

    # -- execution
    def _run(self, steps, exact: bool) -> list[np.ndarray]:
        layout = 0
        sums_per_step = []
        for st in steps:
            if isinstance(st, Swap):
                self._swap(st.nv)
                layout ^= 1
                sums_per_step.append(None)
                continue
            per = []
            for k in range(len(self.ranks)):
                out = (C.c_double * 3)()
                table = self.tables[layout][k]
                call("qsb_layer_sweeps", self.ctx.device.handle, table.table.ptr, self.ket[k].ptr,
                     self.bra[k].ptr if st.nv == 2 else None, st.nv, self.n_l, self.n, st.lo, st.hi, float(st.theta),
                     st.flags | (EXACT if exact else 0), float(st.phase), out)
                per.append(np.array(out[:3]))
            sums_per_step.append(per)
        # one combine for the whole walk: stack every step's per-shard sums
        idx = [i for i, s in enumerate(sums_per_step) if s is not None]
        stacked = [np.concatenate([sums_per_step[i][k] for i in idx]) for k in range(len(self.ranks))]
        total = self.ex.combine(stacked) if stacked else np.zeros(0)
        out = [None] * len(steps)
        for j, i in enumerate(idx):
            out[i] = total[3 * j: 3 * j + 3]
        self.layout = layout
        return out

    def _use_chain(self, exact: bool) -> bool:
        import os

        return not exact and self.n_l >= 21 and os.environ.get("QSB_SHARD_CHAIN", "1") != "0"

    def _run_chain(self, visits: list[Visit]) -> list[np.ndarray]:
        """Execute the window chain on this process's shards (fast mode)."""
        h = self.ctx.device.handle
        layout = self.layout
        per_visit = []
        for v in visits:
            fused = v.swap and self.ex.fused
            if fused and v.nv == 2 and self.scratch_bra is None:
                self.scratch_bra = [DeviceArray(self.ctx.device, 1 << self.n_l, np.complex128) for _ in self.ranks]
            per = []
            for k, r in enumerate(self.ranks):
                d = _ShardVisit(v.nv, v.mode, v.window, v.lo1, v.hi1, v.theta1, v.lo2, v.hi2, v.theta2, v.flags,
                                v.phase, self.g if fused else 0, r)
                if fused:
                    for c, ptr in enumerate(self.ex.targets("ket", self.scratch)):
                        d.out0[c] = ptr
                    if v.nv == 2:
                        for c, ptr in enumerate(self.ex.targets("bra", self.scratch_bra)):
                            d.out1[c] = ptr
                out = (C.c_double * 4)()
                call("qsb_shard_visit_run", h, self.tables[layout][k].table.ptr, self.ket[k].ptr,
                     self.bra[k].ptr if v.nv == 2 else None, self.n_l, self.n, C.byref(d), out)
                per.append(np.array(out[:4]))
            per_visit.append(per)
            if v.swap:
                if fused:
                    self.ex.commit("ket", self.ket, self.scratch)
                    if v.nv == 2:
                        self.ex.commit("bra", self.bra, self.scratch_bra)
                else:
                    self._swap(v.nv)
                layout ^= 1
        stacked = [np.concatenate([pv[k] for pv in per_visit]) for k in range(len(self.ranks))]
        total = self.ex.combine(stacked)
        self.layout = layout
        return [total[4 * j: 4 * j + 4] for j in range(len(visits))]

    def value_and_grad(self, params: circuit.QaoaParams, exact: bool = False):
        if params.p < 1:
            raise ContractViolation("gradient needs depth p >= 1")
        self._plus_pending = False
        if self._use_chain(exact):
            visits = chain_program(self.n, self.g, params.gammas, params.betas, True, True)
            value, dg, db = collect_chain(visits, self._run_chain(visits), params.p)
        else:
            steps = program(self.n, self.g, params.gammas, params.betas, True, True)
            value, dg, db = collect(steps, self._run(steps, exact), params.p)
        # the walk's last sweep only contracts: the ket is |+> by contract (adjoint.py:39-42)
        self._plus_pending = True
        return self._clamp(value), dg, db

    def expectation(self, params: circuit.QaoaParams, exact: bool = False) -> float:
        if params.p < 1:
            raise ContractViolation("sharded expectation needs p >= 1")
        self._plus_pending = False
        if self._use_chain(exact):
            visits = chain_program(self.n, self.g, params.gammas, params.betas, True, False)
            value, _, _ = collect_chain(visits, self._run_chain(visits), params.p)
            return self._clamp(value)
        steps = program(self.n, self.g, params.gammas, params.betas, True, False)
        value, _, _ = collect(steps, self._run(steps, exact), params.p)
        return self._clamp(value)

    def _clamp(self, v: float) -> float:
        return min(max(v, self.min_value), self.max_value)

    def _materialize(self) -> None:
        """write a pending |+> (1/sqrt(2^n) on every shard, layout-independent)"""
        if self._plus_pending:
            amp = 1.0 / np.sqrt(float(1 << self.n))
            for k in range(len(self.ranks)):
                call("qsb_fill_const", self.ctx.device.handle, self.ket[k].ptr, 1 << self.n_l, amp, 0.0)
            self.layout = 0
            self._plus_pending = False

    def gather_state(self) -> np.ndarray:
        """Full statevector in global index order (virtual shards, tests)."""
        if not isinstance(self.ex, VirtualExchanger):
            raise ContractViolation("gather_state needs all shards in this process")
        self._materialize()
        out = np.empty(1 << self.n, dtype=np.complex128)
        i = np.arange(1 << self.n_l, dtype=np.int64)
        for k, r in enumerate(self.ranks):
            out[global_index(self.layout, self.n, self.g, r, i)] = self.ket[k].to_host()
        return out

    def local_state(self) -> tuple[np.ndarray, np.ndarray]:
        """(global indices, amplitudes) of this process's shard(s) in the current layout."""
        self._materialize()
        i = np.arange(1 << self.n_l, dtype=np.int64)
        idx = np.concatenate([global_index(self.layout, self.n, self.g, r, i) for r in self.ranks])
        amps = np.concatenate([self.ket[k].to_host() for k in range(len(self.ranks))])
        return idx, amps

    def draw(self, shots: int, seed: int) -> "sampling.SampleSet":
        """Sample the sharded state (sampling.draw semantics: indices in draw order, the
        reference's probability-tree association and splitmix64 uniforms, so the
        indices equal those of the unsharded state's draw).

        The state first returns to layout A (rank bits = top index bits) with a
        standalone swap when an odd number of swaps preceded.  Shards build their
        subtrees on their GPUs (qsb_sample_tree); the G roots are gathered and combined
        pairwise exactly like the reference's upper tree levels; every rank draws
        u_s = U(seed, s) * total and descends those g levels (identical arithmetic
        everywhere), then each shard descends its own shots on the device
        (qsb_sample_descend) and the per-shot results are summed over ranks (one owner
        per shot)."""
        if shots < 1:
            raise ContractViolation(f"shots must be >= 1, got {shots}")
        self._materialize()
        if self.layout != 0:  # back to layout A: the rank bits are the top index bits
            self._swap(1)
            self.layout = 0
        h = self.ctx.device.handle
        local = []
        for k in range(len(self.ranks)):
            r = C.c_double()
            call("qsb_sample_tree", h, self.ket[k].ptr, self.n_l, C.byref(r))
            local.append(r.value)
        levels = [np.asarray(self.ex.gather(local), dtype=np.float64)]  # level n_l .. n
        while levels[-1].shape[0] > 1:
            v = levels[-1]
            levels.append(v[0::2] + v[1::2])
        total = float(levels[-1][0])
        if not abs(total - 1.0) <= 1e-9:
            raise ContractViolation(f"state is not normalized: sum of probabilities = {total!r}")
        u = rng.uniform_block(seed, 0, shots) * total
        shard = np.zeros(shots, dtype=np.int64)
        for j in range(self.g - 1, -1, -1):
            left = levels[j][2 * shard]
            right = u >= left
            u = np.where(right, u - left, u)
            shard = 2 * shard + right
        idx = np.zeros(shots, dtype=np.int64)
        cost = np.zeros(shots, dtype=np.float64)
        for k, r in enumerate(self.ranks):
            sel = np.flatnonzero(shard == r)
            if sel.size == 0:
                continue
            if len(self.ranks) > 1:  # virtual shards share one context: rebuild this shard's tree
                r_ = C.c_double()
                call("qsb_sample_tree", h, self.ket[k].ptr, self.n_l, C.byref(r_))
            ui = np.ascontiguousarray(u[sel])
            li = np.empty(sel.size, dtype=np.int64)
            ci = np.empty(sel.size, dtype=np.float64)
            call("qsb_sample_descend", h, self.tables[0][k].table.ptr, self.ket[k].ptr, self.n_l, int(sel.size),
                 ui.ctypes.data, li.ctypes.data, ci.ctypes.data)
            idx[sel] = li | (int(r) << self.n_l)
            cost[sel] = ci
        idx, cost = self.ex.owned_sum(idx, cost)
        return sampling.SampleSet(shots=shots, seed=seed, indices=idx, costs=cost)

    def simulate(self, params: circuit.QaoaParams, exact: bool = False) -> None:
        self._plus_pending = False
        if self._use_chain(exact) and params.p >= 1:
            self._run_chain(chain_program(self.n, self.g, params.gammas, params.betas, False, False))
            return
        steps = program(self.n, self.g, params.gammas, params.betas, False, False)
        self._run(steps, exact)

    def memory_bytes(self) -> int:
        """device bytes this process holds for the handle (statevectors + tables)"""
        N_l = 1 << self.n_l
        nvec = 3 + (1 if self.scratch_bra is not None else 0)
        return len(self.ranks) * nvec * 16 * N_l + self.table_bytes

    def close(self) -> None:
        if hasattr(self.ex, "close"):
            self.ex.close()
        for arrs in (self.ket, self.bra, self.scratch, self.scratch_bra or [], *self.tables):
            for a in arrs:
                a.free()
