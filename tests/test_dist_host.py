"""Sharded path, host side (no GPU): the layout maps, the index-bit swap and the
whole sharded schedule (dist.program + dist.collect) executed by a numpy emulator
on shards, against the dense oracle; plus the one-shard-per-process exchange over
torch.distributed (gloo, world_size 2) reproducing the virtual-shard permutation."""

import math
import os
import socket

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import dist

from conftest import random_instance, random_params
from oracle import oracle


@pytest.mark.parametrize("n,g", [(5, 1), (6, 2), (7, 3), (12, 2)])
def test_layouts_are_bijections(n, g):
    i = np.arange(1 << (n - g))
    for layout in (0, 1):
        xs = np.concatenate([dist.global_index(layout, n, g, r, i) for r in range(1 << g)])
        assert sorted(xs.tolist()) == list(range(1 << n))


def emulate_swap(shards, G):
    chunk = len(shards[0]) // G
    out = [np.empty_like(s) for s in shards]
    for r in range(G):
        for c in range(G):
            out[c][r * chunk:(r + 1) * chunk] = shards[r][c * chunk:(c + 1) * chunk]
    return out


@pytest.mark.parametrize("n,g", [(6, 1), (8, 2), (9, 3)])
def test_swap_maps_layout_a_to_b_and_back(n, g):
    G = 1 << g
    psi = np.random.default_rng(n).normal(size=1 << n) + 0j
    i = np.arange(1 << (n - g))
    a = [psi[dist.global_index(0, n, g, r, i)] for r in range(G)]
    b = emulate_swap(a, G)
    for r in range(G):
        assert np.array_equal(b[r], psi[dist.global_index(1, n, g, r, i)])
    back = emulate_swap(b, G)
    for r in range(G):
        assert np.array_equal(back[r], a[r])


class Emulator:
    """Executes dist.program() on numpy shards with the oracle's per-qubit kernels."""

    def __init__(self, poly, g):
        self.n, self.g, self.n_l = poly.n, g, poly.n - g
        self.G = 1 << g
        full = oracle.precompute_table(poly.weights, poly.masks, poly.n)
        i = np.arange(1 << self.n_l)
        self.tables = [[np.ascontiguousarray(full[dist.global_index(L, self.n, g, r, i)]) for r in range(self.G)]
                       for L in (0, 1)]

    def run(self, steps):
        G, n_l = self.G, self.n_l
        ket = [np.empty(1 << n_l, complex) for _ in range(G)]
        bra = [np.empty(1 << n_l, complex) for _ in range(G)]
        layout, out = 0, []
        for st in steps:
            if isinstance(st, dist.Swap):
                ket = emulate_swap(ket, G)
                if st.nv == 2:
                    bra = emulate_swap(bra, G)
                layout ^= 1
                out.append(None)
                continue
            tot = np.zeros(3)
            c, s = math.cos(st.theta / 2.0), math.sin(st.theta / 2.0)
            for r in range(G):
                t = self.tables[layout][r]
                k, b = ket[r], bra[r]
                if st.flags & dist.PLUS:
                    k[:] = 1.0 / math.sqrt(1 << self.n)
                if st.flags & dist.BRA_FROM_KET:
                    b[:] = t * k
                if st.flags & dist.PRE_DINNER:
                    tot[1] += np.sum(t * (np.conj(b) * k).imag)
                if st.flags & dist.PRE_PHASE:
                    f = np.exp(1j * st.phase * t)
                    k *= f
                    if st.nv == 2:
                        b *= f
                idx = np.arange(1 << n_l)
                for j in range(st.lo, st.hi + 1):
                    if st.flags & dist.XSUM:
                        tot[2] += np.sum((np.conj(b) * k[idx ^ (1 << j)]).imag)
                    oracle.rx_qubit(k, j, c, s)
                    if st.nv == 2:
                        oracle.rx_qubit(b, j, c, s)
                if st.flags & dist.POST_EXPECT:
                    tot[0] += np.sum(t * np.abs(k) ** 2)
                if st.flags & dist.POST_DINNER:
                    tot[0] += np.sum(t * (np.conj(b) * k).imag)
            out.append(tot)
        self.layout, self.ket = layout, ket
        return out


@pytest.mark.parametrize("n,g,p,seed", [(6, 1, 1, 1), (7, 2, 2, 2), (8, 3, 3, 3), (9, 1, 4, 4)])
def test_sharded_schedule_matches_dense_oracle(n, g, p, seed):
    poly = random_instance(seed * 11 + 5, n)
    params = random_params(seed + 40, p)
    em = Emulator(poly, g)
    steps = dist.program(n, g, params.gammas, params.betas, True, True)
    value, dg, db = dist.collect(steps, em.run(steps), p)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, wdg, wdb = oracle.value_and_grad(table, n, params.gammas, params.betas)
    assert abs(value - e) <= 1e-12 * max(1, abs(e))
    assert np.max(np.abs(np.concatenate([dg - wdg, db - wdb]))) <= 1e-11 * max(1, np.max(np.abs(wdb)))


def test_sharded_forward_state_matches_dense(n=8, g=2):
    poly = random_instance(3, n)
    params = random_params(9, 3)
    em = Emulator(poly, g)
    em.run(dist.program(n, g, params.gammas, params.betas, False, False))
    full = np.empty(1 << n, complex)
    i = np.arange(1 << (n - g))
    for r in range(1 << g):
        full[dist.global_index(em.layout, n, g, r, i)] = em.ket[r]
    want = oracle.simulate(oracle.precompute_table(poly.weights, poly.masks, n), n, params.gammas, params.betas)
    assert np.max(np.abs(full - want)) < 1e-13


def _gloo_worker(rank, world, port, n, g, q):
    import torch
    import torch.distributed as tdist

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    psi = np.arange(1 << n, dtype=np.float64) * 1.5 + 0.25
    i = np.arange(1 << (n - g))
    mine = torch.tensor(psi[dist.global_index(0, n, g, rank, i)]).view(world, -1)
    out = torch.empty_like(mine)
    tdist.all_to_all_single(out, mine)  # the TorchExchanger.swap collective
    ok = np.array_equal(out.view(-1).numpy(), psi[dist.global_index(1, n, g, rank, i)])
    tdist.destroy_process_group()
    q.put((rank, ok))


def test_all_to_all_over_gloo_is_the_layout_swap():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, 8, 1, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


class _HostArr:
    """host stand-in for a DeviceArray: memory addressed by .ptr (so pointer swaps
    behave like the device buffers')"""

    store: dict = {}

    def __init__(self, values):
        self.ptr = len(_HostArr.store) + 1000
        _HostArr.store[self.ptr] = np.array(values, dtype=np.complex128)

    def __len__(self):
        return len(_HostArr.store[self.ptr])

    def to_host(self):
        return _HostArr.store[self.ptr].copy()

    def from_host(self, values):
        _HostArr.store[self.ptr][:] = values


def _staged_swap_worker(rank, world, port, n, g, q):
    import torch.distributed as tdist

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        psi = (np.arange(1 << n, dtype=np.float64) * 1.5 + 0.25) * (1 - 0.5j)
        i = np.arange(1 << (n - g))
        ex = dist.TorchExchanger(g, tdist, 0, p2p=False)
        live = [_HostArr(psi[dist.global_index(0, n, g, rank, i)])]
        spare = [_HostArr(np.zeros(1 << (n - g)))]
        ex.swap_vec("ket", live, spare)  # the non-P2P branch over gloo: staged through the host
        ok = np.array_equal(live[0].to_host(), psi[dist.global_index(1, n, g, rank, i)])
        ex.swap_vec("ket", live, spare)  # and back
        ok = ok and np.array_equal(live[0].to_host(), psi[dist.global_index(0, n, g, rank, i)])
    finally:
        tdist.destroy_process_group()
    q.put((rank, bool(ok)))


def _p2p_setup_worker(rank, world, port, q):
    """rank 0 exports its IPC handles, rank 1 fails to: both must still run the same
    collectives and agree to fall back (no mismatched all_gather / all_reduce hang)"""
    import torch.distributed as tdist

    from paper_2407_13012_b200 import _lib

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        def fake_call(name, *args):
            if rank == 1 or name != "qsb_ipc_handle":
                raise _lib.ContractViolation(f"{name}: no peer access on rank {rank}")

        dist.call = fake_call

        class _Dev:
            handle = None

        class _Ctx:
            device = _Dev()

        class _H:
            ctx = _Ctx()
            ket = [_HostArr(np.zeros(4))]
            scratch = [_HostArr(np.zeros(4))]
            bra = [_HostArr(np.zeros(4))]
            scratch_bra = [_HostArr(np.zeros(4))]

        ex = dist.TorchExchanger(1, tdist, 0, p2p=True)
        ex.setup(_H())
        q.put((rank, ex.fused))
    finally:
        tdist.destroy_process_group()


def _spawn(target, args_of_rank, world=2):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, *args_of_rank(r), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def test_torch_exchanger_staged_swap_over_gloo():
    """TorchExchanger.swap_vec without P2P on a gloo group: D2H, all_to_all_single of
    host tensors, H2D into the spare, pointer swap -- layout A <-> B exactly"""
    assert _spawn(_staged_swap_worker, lambda r: (9, 1)) == {0: True, 1: True}


def test_p2p_setup_failure_on_one_rank_falls_back_everywhere():
    assert _spawn(_p2p_setup_worker, lambda r: ()) == {0: False, 1: False}


def _nccl_setup_worker(rank, world, port, fail_rank, q):
    """libqsb's NCCL communicator setup (TorchExchanger._setup_nccl) with the library
    calls faked: rank 0's unique id is broadcast, every rank initialises, and one
    all_reduce decides -- a rank whose init fails makes every rank stay on torch's
    all-to-all (and the ranks that did initialise destroy their communicators)"""
    import ctypes as C

    import torch.distributed as tdist

    from paper_2407_13012_b200 import _lib

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    destroyed = []
    seen_id = []
    try:
        def fake_call(name, *args):
            if name == "qsb_nccl_unique_id":
                C.memmove(args[0], bytes(range(7, 135)), 128)
            elif name == "qsb_nccl_init":
                seen_id.append(C.string_at(args[1], 128) == bytes(range(7, 135)))
                if rank == fail_rank:
                    raise _lib.ContractViolation("ncclCommInitRank: no")
                args[4]._obj.value = 4096 + rank
            elif name == "qsb_nccl_destroy":
                destroyed.append(args[0])

        dist.call = fake_call

        class _Dev:
            handle = None

        class _Ctx:
            device = _Dev()

        class _H:
            ctx = _Ctx()

        ex = dist.TorchExchanger(1, tdist, 0, p2p=False)
        ex._setup_nccl(_H(), force=True)
        q.put((rank, (ex._nccl, destroyed, seen_id == [True])))
    finally:
        tdist.destroy_process_group()


def test_native_nccl_setup_agrees_across_ranks():
    assert _spawn(_nccl_setup_worker, lambda r: (-1,)) == {0: (4096, [], True), 1: (4097, [], True)}
    assert _spawn(_nccl_setup_worker, lambda r: (1,)) == {0: (None, [4096], True), 1: (None, [], True)}


def test_nccl_library_is_reachable():
    """libqsb opens libnccl.so.2 at run time (the copy torch loaded): version and a
    unique id work without a GPU; bad arguments are contract violations"""
    import ctypes as C

    import torch  # noqa: F401  (loads torch's NCCL first, as in a real run)

    from paper_2407_13012_b200 import _lib

    v = C.c_int32()
    _lib.call("qsb_nccl_version", C.byref(v))
    assert v.value >= 22700
    uid = np.zeros(128, dtype=np.uint8)
    _lib.call("qsb_nccl_unique_id", uid.ctypes.data)
    assert uid.any()
    with pytest.raises(_lib.ContractViolation):
        _lib.call("qsb_nccl_init", None, uid.ctypes.data, 2, 0, C.byref(C.c_void_p()))
    with pytest.raises(_lib.ContractViolation):
        _lib.call("qsb_nccl_all_to_all", None, None, None, 0)
