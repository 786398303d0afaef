"""Sharded path on one B200 with virtual shards (the all-to-all becomes device
copies): same kernels and schedule as the multi-GPU run, checked against the
unsharded fused path and the CPU oracle."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import dist

from conftest import random_instance, random_params, rel_err
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,g,p,seed", [(14, 1, 2, 1), (15, 2, 3, 2), (16, 3, 2, 3), (20, 2, 4, 4), (22, 1, 3, 5)])
def test_sharded_value_and_grad(n, g, p, seed):
    poly = random_instance(seed * 7 + 1, n)
    params = random_params(seed + 100, p)
    sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
    value, dg, db = sh.value_and_grad(params)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, wdg, wdb = oracle.value_and_grad(table, n, params.gammas, params.betas)
    assert abs(value - e) <= 1e-10 * max(1.0, abs(e))
    assert rel_err(np.concatenate([dg, db]), np.concatenate([wdg, wdb])) <= 1e-10
    # unsharded fused path on the same device agrees too
    h = qs.create_handle(poly, backend_name="b200")
    v1, g1 = qs.value_and_grad(h, params)
    assert abs(v1 - value) <= 1e-10 * max(1.0, abs(e))
    sh.close()
    h.close()


@pytest.mark.parametrize("n,g", [(14, 2), (17, 1)])
def test_sharded_statevector_and_expectation(n, g):
    poly = random_instance(n, n)
    params = random_params(n + 1, 3)
    sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
    e = sh.expectation(params)
    psi = sh.gather_state()
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    want = oracle.simulate(table, n, params.gammas, params.betas)
    assert rel_err(psi, want) <= 1e-10
    assert abs(e - oracle.expectation(table, want)) <= 1e-10 * max(1.0, abs(e))
    assert (sh.min_value, sh.max_value) == (table.min(), table.max())
    sh.close()


def test_sharded_weighted_and_float_tables():
    # integer weights (u16 compact index) and a float QUBO (f64 table + device sincos)
    from paper_2407_13012_b200 import rng

    s = rng.Stream(5)
    n = 14
    edges = [(u, v, float(1 + int(300 * s.next_uniform()))) for u in range(n) for v in range(u + 1, n)]
    wpoly = qs.maxcut_polynomial(qs.Graph(n, edges))
    qterms = [((s.next_uniform() - 0.5) * 8, (1 << i) | (1 << j)) for i in range(n) for j in range(i, n)]
    qpoly = qs.Polynomial(n, qterms)
    params = random_params(77, 2)
    for poly in (wpoly, qpoly):
        sh = dist.ShardedHandle(poly, 2, dist.VirtualExchanger(2))
        value, dg, db = sh.value_and_grad(params)
        table = oracle.precompute_table(poly.weights, poly.masks, n)
        e, wdg, wdb = oracle.value_and_grad(table, n, params.gammas, params.betas)
        assert abs(value - e) <= 1e-10 * max(1.0, abs(e))
        assert rel_err(np.concatenate([dg, db]), np.concatenate([wdg, wdb])) <= 1e-10
        sh.close()


@pytest.mark.parametrize("n,g", [(14, 1), (15, 2), (16, 3)])
def test_sharded_draw_matches_the_unsharded_tree(n, g):
    """sharded sampling: the same indices and costs as the reference's draw on the
    gathered state (same tree association, same uniforms)"""
    poly = random_instance(40 + n, n)
    params = random_params(n + 5, 2)
    sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
    sh.simulate(params)
    state = sh.gather_state()
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    ss = sh.draw(20000, 11)
    idx, cost = oracle.sample(state, table, 20000, 11)
    assert np.array_equal(ss.indices, idx)
    assert np.array_equal(ss.costs, cost)
    assert sh.layout == 0
    sh.close()


@pytest.mark.parametrize("n,g,p", [(22, 1, 2), (23, 2, 3), (24, 3, 2), (26, 1, 1)])
def test_sharded_window_chain(n, g, p, monkeypatch):
    """fast-mode sharded walk as a window chain (dist.chain_program): merged visits at
    the top window, the qubit swap fused into the A visit's stores (virtual shards:
    stores straight into the other shards' buffers) -- against the per-position
    schedule (QSB_SHARD_CHAIN=0) and the unsharded single-GPU chain"""
    poly = random_instance(60 + n, n)
    params = random_params(n + 9, p)
    sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
    v1, dg1, db1 = sh.value_and_grad(params)
    e1 = sh.expectation(params)
    sh.simulate(params)
    st1 = sh.gather_state()
    monkeypatch.setenv("QSB_SHARD_CHAIN", "0")
    v0, dg0, db0 = sh.value_and_grad(params)
    sh.simulate(params)
    st0 = sh.gather_state()
    sh.close()
    h = qs.create_handle(poly, backend_name="b200")
    v2, g2 = qs.value_and_grad(h, params)
    h.close()
    assert abs(v1 - v0) <= 1e-11 * max(1.0, abs(v0)) and abs(v1 - v2) <= 1e-11 * max(1.0, abs(v2))
    assert abs(e1 - v1) <= 1e-11 * max(1.0, abs(v1))
    ref = np.concatenate([np.array(g2.d_gammas), np.array(g2.d_betas)])
    assert rel_err(np.concatenate([dg1, db1]), ref) <= 1e-10
    assert rel_err(np.concatenate([dg1, db1]), np.concatenate([dg0, db0])) <= 1e-11
    assert rel_err(st1, st0) <= 1e-12


@pytest.mark.parametrize("mode", ["p2p", "staged", "nccl"])
@pytest.mark.parametrize("n,p", [(22, 3), (16, 3)])
def test_two_process_sharded(tmp_path, mode, n, p):
    """Two processes, one shard each (both on the one GPU here), for both transports
    of dist.TorchExchanger: "p2p" (qubit swap fused into the A visit's stores through
    CUDA IPC; standalone swaps by the peer chunk scatter), "staged" (the all-to-all
    branch, host-staged over gloo) and "nccl" (the all-to-all on libqsb's own NCCL
    communicator; host collectives still over gloo).  n=22: the window chain (n_l = 21); n=16: the
    per-position schedule (n_l < 21: every swap standalone).  Fast and exact
    value_and_grad, a draw after an odd number of layers (layout B -> swap back) and a
    draw after a gradient (ket |+> by contract) equal the single-process virtual-shard
    run and the CPU oracle."""
    import os
    import subprocess
    import sys

    out = tmp_path / "res.npz"
    port = 29531 + (n % 7) * 3 + ["staged", "p2p", "nccl"].index(mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(os.path.dirname(__file__), "mp_shard_worker.py"), str(out), str(n), str(p), mode]
    res = subprocess.run(cmd, env=dict(os.environ), capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    got = np.load(out)
    if mode == "nccl" and not int(got["native"]):
        pytest.skip("NCCL would not initialise two ranks on one GPU (both fell back to the staged swap)")
    assert int(got["fused"]) == (1 if mode == "p2p" else 0)
    assert int(got["layout"]) == p % 2  # one swap per layer: odd p ends in layout B
    poly = random_instance(70 + n, n)
    params = random_params(n + 3, p)
    sh = dist.ShardedHandle(poly, 1, dist.VirtualExchanger(1))
    v, dg, db = sh.value_and_grad(params)
    vx, dgx, dbx = sh.value_and_grad(params, exact=True)
    sh.simulate(params)
    state = sh.gather_state()
    sh.close()
    assert abs(float(got["v"]) - v) <= 1e-12 * max(1.0, abs(v))
    assert abs(float(got["e"]) - v) <= 1e-11 * max(1.0, abs(v))
    assert rel_err(np.concatenate([got["dg"], got["db"]]), np.concatenate([dg, db])) <= 1e-12
    assert float(got["vx"]) == vx
    assert np.array_equal(got["dgx"], dgx) and np.array_equal(got["dbx"], dbx)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, wdg, wdb = oracle.value_and_grad(table, n, params.gammas, params.betas)
    assert abs(v - e) <= 1e-10 * max(1.0, abs(e))
    assert rel_err(np.concatenate([dgx, dbx]), np.concatenate([wdg, wdb])) <= 1e-10
    idx, cost = oracle.sample(state, table, 4000, 11)
    assert np.array_equal(got["idx"], idx) and np.array_equal(got["cost"], cost)
    plus = np.full(1 << n, 1.0 / np.sqrt(float(1 << n)), dtype=np.complex128)
    gidx, gcost = oracle.sample(plus, table, 3000, 5)
    assert np.array_equal(got["gidx"], gidx) and np.array_equal(got["gcost"], gcost)


def test_sharded_chain_float_table_and_sampling():
    """window chain with an f64 table (device sincos between the passes) and a draw
    from the chain-simulated sharded state"""
    n, g, p = 22, 1, 2
    rs = np.random.default_rng(5)
    terms = [((rs.random() - 0.5) * 6.0, 1 << i) for i in range(n)]
    terms += [((rs.random() - 0.5) * 6.0, (1 << i) | (1 << j)) for i in range(n) for j in range(i + 1, n)
              if rs.random() < 0.3]
    poly = qs.Polynomial(n, terms)
    params = random_params(12, p)
    sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
    v, dg, db = sh.value_and_grad(params)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, wdg, wdb = oracle.value_and_grad(table, n, params.gammas, params.betas)
    assert abs(v - e) <= 1e-10 * max(1.0, abs(e))
    assert rel_err(np.concatenate([dg, db]), np.concatenate([wdg, wdb])) <= 1e-10
    sh.simulate(params)
    state = sh.gather_state()
    ss = sh.draw(5000, 3)
    idx, cost = oracle.sample(state, table, 5000, 3)
    assert np.array_equal(ss.indices, idx) and np.array_equal(ss.costs, cost)
    sh.close()


def test_native_nccl_all_to_all_single_rank():
    """libqsb's NCCL transport on the GPU, one rank: the group of send/recv pairs on
    the context stream moves the chunk, stream-ordered after the H2D and before the D2H
    (two ranks: test_two_process_sharded's "nccl" mode)"""
    import ctypes as C

    import torch  # noqa: F401  (torch's NCCL is the one libqsb opens)

    from paper_2407_13012_b200 import _lib
    from paper_2407_13012_b200._lib import DeviceArray, DeviceContext, call

    dctx = DeviceContext(0)
    rs = np.random.default_rng(4)
    x = rs.standard_normal(1 << 16) + 1j * rs.standard_normal(1 << 16)
    src = DeviceArray(dctx, len(x), np.complex128)
    dst = DeviceArray(dctx, len(x), np.complex128)
    src.from_host(x)
    uid = np.zeros(128, dtype=np.uint8)
    call("qsb_nccl_unique_id", uid.ctypes.data)
    comm = C.c_void_p()
    call("qsb_nccl_init", dctx.handle, uid.ctypes.data, 1, 0, C.byref(comm))
    try:
        call("qsb_nccl_all_to_all", comm, src.ptr, dst.ptr, len(x))
        call("qsb_nccl_wait", comm, 60000)  # completes: no async error, within the timeout
        assert np.array_equal(dst.to_host(), x)
    finally:
        call("qsb_nccl_destroy", comm)
    with pytest.raises(_lib.ContractViolation):
        call("qsb_nccl_init", dctx.handle, uid.ctypes.data, 1, 1, C.byref(C.c_void_p()))
