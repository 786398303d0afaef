"""Z2 reduction (flip-symmetric cost tables: every MaxCut): the fused chains evolve
only x < 2^(n-1) (psi(x) = psi(~x)), the A window on tile pairs {T, ~T}.  Checked
against the CPU oracle and against the full (QSB_NO_SYM=1) fast path."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200.kernels import b200

from conftest import random_instance, random_params, rel_err
from oracle import oracle

pytestmark = pytest.mark.gpu


def test_symmetry_detection():
    h = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(22, 3, seed=1)), backend_name="b200")
    assert b200.table_symmetric(h.table.values.data, 22)
    qubo = qs.Polynomial(22, [(0.5, 1 << 3), (1.25, (1 << 4) | (1 << 9))])
    h2 = qs.create_handle(qubo, backend_name="b200")
    assert not b200.table_symmetric(h2.table.values.data, 22)
    h.close()
    h2.close()


@pytest.mark.parametrize("n,p,seed", [(21, 3, 1), (22, 1, 2), (23, 4, 3), (24, 2, 4), (26, 3, 5)])
def test_reduced_chain_vs_oracle_and_full(n, p, seed, monkeypatch):
    poly = random_instance(900 + seed, n)
    params = random_params(seed, p)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, dg, db = oracle.value_and_grad(table, n, params.gammas, params.betas)
    psi = oracle.simulate(table, n, params.gammas, params.betas)
    h = qs.create_handle(poly, backend_name="b200")
    assert b200.table_symmetric(h.table.values.data, n)
    v, g = qs.value_and_grad(h, params)
    assert abs(v - e) <= 1e-10 * max(1.0, abs(e))
    got = np.concatenate([g.d_gammas, g.d_betas])
    assert rel_err(got, np.concatenate([dg, db])) <= 1e-10
    ev = qs.expectation(h, params)
    assert abs(ev - e) <= 1e-10 * max(1.0, abs(e))
    st = qs.statevector(h, params)  # the mirror half is written on this read
    assert rel_err(st, psi) <= 1e-10
    assert np.array_equal(st[: 1 << (n - 1)], st[::-1][: 1 << (n - 1)])  # psi(x) == psi(~x) bit for bit
    qs.simulate(h, params)
    ss = qs.draw(h, 3000, 9)
    idx, cost = oracle.sample(np.asarray(h.state.data), table, 3000, 9)
    assert np.array_equal(ss.indices, idx) and np.array_equal(ss.costs, cost)
    monkeypatch.setenv("QSB_NO_SYM", "1")
    v1, g1 = qs.value_and_grad(h, params)
    assert abs(v1 - v) <= 1e-12 * max(1.0, abs(v))
    assert rel_err(np.concatenate([g1.d_gammas, g1.d_betas]), got) <= 1e-12
    h.close()


@pytest.mark.parametrize("n,p,seed", [(21, 2, 11), (24, 3, 12)])
def test_half_state_sampling(n, p, seed, monkeypatch):
    """Draws from the lower half of a Z2-reduced state (qsb_sample_sym: no mirror copy,
    half the tree) are the draws of the materialised state, bit for bit."""
    poly = random_instance(700 + seed, n)
    params = random_params(seed, p)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    h = qs.create_handle(poly, backend_name="b200")
    qs.simulate(h, params)
    assert h.state.half_view() is not None  # the upper half is still unwritten
    ss = qs.draw(h, 50000, seed)
    assert h.state.half_view() is not None  # drawn from the half
    assert (ss.indices >= (1 << (n - 1))).any() and (ss.indices < (1 << (n - 1))).any()
    monkeypatch.setenv("QSB_NO_HALF_SAMPLE", "1")
    full = qs.draw(h, 50000, seed)  # materialises the mirror, full tree
    assert h.state.half_view() is None
    assert np.array_equal(ss.indices, full.indices) and np.array_equal(ss.costs, full.costs)
    idx, cost = oracle.sample(np.asarray(h.state.data), table, 50000, seed)
    assert np.array_equal(ss.indices, idx) and np.array_equal(ss.costs, cost)
    h.close()


def test_reduced_batch_many():
    from paper_2407_13012_b200 import batch

    polys = [random_instance(950 + k, 21 + k % 2) for k in range(4)]
    params = [random_params(60 + k, 2) for k in range(4)]
    hs = [qs.create_handle(pl, backend_name="b200") for pl in polys]
    got = batch.value_and_grad_batch(hs, params)
    for pl, prm, (v, g) in zip(polys, params, got):
        table = oracle.precompute_table(pl.weights, pl.masks, pl.n)
        e, dg, db = oracle.value_and_grad(table, pl.n, prm.gammas, prm.betas)
        assert abs(v - min(max(e, table.min()), table.max())) <= 1e-10 * max(1.0, abs(e))
        assert rel_err(np.concatenate([g.d_gammas, g.d_betas]), np.concatenate([dg, db])) <= 1e-10
    for h in hs:
        h.close()


@pytest.mark.parametrize("n,p,sym", [(22, 3, True), (23, 2, False), (16, 4, True)])
def test_forward_checkpoints(n, p, sym, monkeypatch):
    """the adjoint walk with forward checkpoints in spare HBM (backward sweeps read the
    ket from them and never store it) equals the in-place walk and the oracle"""
    if sym:
        poly = random_instance(1200 + n, n)
    else:  # a QUBO-like table with linear terms: not flip-symmetric
        rs = np.random.default_rng(n)
        poly = qs.Polynomial(n, [((rs.random() - 0.5) * 4, 1 << i) for i in range(n)] +
                             [((rs.random() - 0.5) * 4, (1 << i) | (1 << ((i + 3) % n))) for i in range(n)])
    params = random_params(77 + n, p)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    e, dg, db = oracle.value_and_grad(table, n, params.gammas, params.betas)
    h = qs.create_handle(poly, backend_name="b200")
    v, g = qs.value_and_grad(h, params)  # checkpoints (default)
    monkeypatch.setenv("QSB_NO_CKPT", "1")
    v0, g0 = qs.value_and_grad(h, params)
    monkeypatch.delenv("QSB_NO_CKPT")
    monkeypatch.setenv("QSB_CKPT_MARGIN_GB", "170")  # no room: in place
    v1, g1 = qs.value_and_grad(h, params)
    got = np.concatenate([g.d_gammas, g.d_betas])
    assert abs(v - min(max(e, table.min()), table.max())) <= 1e-10 * max(1.0, abs(e))
    assert rel_err(got, np.concatenate([dg, db])) <= 1e-10
    assert abs(v - v0) <= 1e-12 * max(1.0, abs(v))
    assert rel_err(got, np.concatenate([g0.d_gammas, g0.d_betas])) <= 1e-12
    assert rel_err(got, np.concatenate([g1.d_gammas, g1.d_betas])) <= 1e-12
    # the ket is |+> by contract afterwards
    plus = np.full(1 << n, 1.0 / np.sqrt(float(1 << n)))
    assert np.max(np.abs(np.asarray(h.state.data) - plus)) <= 1e-12
    h.close()


def test_checkpoints_given_back_when_memory_runs_out():
    """checkpoints cached with a context are spare HBM: an allocation that finds the
    device full takes them back (ctx.cu plain_alloc -> release_all_checkpoints) and
    succeeds, and the next gradient rebuilds them with the same result"""
    import ctypes as C

    from paper_2407_13012_b200._lib import call

    n, p = 27, 3
    poly = random_instance(1300 + n, n)
    params = random_params(5, p)
    h = qs.create_handle(poly, backend_name="b200")
    v, g = qs.value_and_grad(h, params)  # leaves >= 3 GiB of checkpoints on h's context
    dev = h.ctx.device
    _, free0, _ = dev.info()
    ptr = C.c_void_p()
    call("qsb_alloc", dev.handle, free0 + (512 << 20), C.byref(ptr))  # more than is free
    try:
        assert ptr.value
    finally:
        call("qsb_free", dev.handle, ptr)
    v2, g2 = qs.value_and_grad(h, params)
    assert v2 == v
    assert np.array_equal(np.asarray(g2.d_gammas), np.asarray(g.d_gammas))
    assert np.array_equal(np.asarray(g2.d_betas), np.asarray(g.d_betas))
    h.close()
