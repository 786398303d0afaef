"""The merged window chain (fused.cu run_chain): consecutive layers meet on the same
window and share one HBM pass (merged / bridge sweeps).  Parity: the chain must
agree with the one-visit-per-sweep schedule (QSB_NO_MERGE=1) to ~1e-12 and with the
CPU oracle (the reference's op sequence) within the north-star 1e-10, across
register sizes whose windows are partial (odd n, n - 12 not a multiple of 9), both
gate forms (|cos| >= |sin| and below) and the float-weight (device sincos) table."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs

from conftest import variant_available, random_instance, random_params, rel_err
from oracle import oracle

pytestmark = pytest.mark.gpu


def flat(g):
    out = np.empty(2 * g.p)
    out[0::2] = g.d_gammas
    out[1::2] = g.d_betas
    return out


def run(poly, params, monkeypatch, merge):
    monkeypatch.setenv("QSB_NO_MERGE", "0" if merge else "1")
    h = qs.create_handle(poly, backend_name="b200")
    v, g = qs.value_and_grad(h, params)
    e = qs.expectation(h, params)
    psi = np.asarray(qs.statevector(h, params))
    h.close()
    return v, flat(g), e, psi


def params_wide(seed, p):
    """angles over (-pi, pi): both factored gate forms occur"""
    rs = np.random.default_rng(seed)
    return qs.QaoaParams(list(rs.uniform(-3.0, 3.0, p)), list(rs.uniform(-1.5, 1.5, p)))


@pytest.mark.parametrize("n,p", [(12, 2), (13, 1), (13, 3), (16, 2), (21, 2), (22, 3), (24, 1)])
def test_chain_vs_oracle(n, p, monkeypatch):
    poly = random_instance(1000 + n * 7 + p, n)
    params = params_wide(n * 31 + p, p)
    v, g, e, psi = run(poly, params, monkeypatch, merge=True)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    want_psi = oracle.simulate(table, n, params.gammas, params.betas)
    want_e = oracle.expectation(table, want_psi)
    dg, db = oracle.gradient(table, want_psi.copy(), params.gammas, params.betas)
    want = np.empty(2 * p)
    want[0::2], want[1::2] = dg, db
    assert abs(v - want_e) <= 1e-10 * max(1.0, abs(want_e))
    assert abs(e - want_e) <= 1e-10 * max(1.0, abs(want_e))
    assert rel_err(g, want) <= 1e-10
    assert rel_err(psi, want_psi) <= 1e-10


@pytest.mark.parametrize("n,p", [(25, 2), (27, 3), (28, 2), (30, 1)])
def test_chain_vs_unmerged(n, p, monkeypatch):
    """3-window registers (partial last window at n = 25, 27, 28) against the
    unmerged schedule on the same GPU"""
    poly = random_instance(77 + n, n)
    params = params_wide(5 * n + p, p)
    got = run(poly, params, monkeypatch, merge=True)
    ref = run(poly, params, monkeypatch, merge=False)
    assert abs(got[0] - ref[0]) <= 1e-12 * max(1.0, abs(ref[0]))
    assert rel_err(got[1], ref[1]) <= 1e-12
    assert abs(got[2] - ref[2]) <= 1e-12 * max(1.0, abs(ref[2]))
    assert rel_err(got[3], ref[3]) <= 1e-12
    assert abs(np.vdot(got[3], got[3]).real - 1.0) <= 1e-10


def test_chain_float_table(monkeypatch):
    """dense QUBO with float weights: f64 table + device sincos inside merged sweeps"""
    n, p = 18, 3
    rs = np.random.default_rng(3)
    terms = [((rs.random() - 0.5) * 8.0, 1 << i) for i in range(n)]
    terms += [((rs.random() - 0.5) * 8.0, (1 << i) | (1 << j)) for i in range(n) for j in range(i + 1, n) if rs.random() < 0.5]
    poly = qs.Polynomial(n, terms)
    params = params_wide(9, p)
    v, g, e, psi = run(poly, params, monkeypatch, merge=True)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    want_psi = oracle.simulate(table, n, params.gammas, params.betas)
    want_e = oracle.expectation(table, want_psi)
    dg, db = oracle.gradient(table, want_psi.copy(), params.gammas, params.betas)
    want = np.empty(2 * p)
    want[0::2], want[1::2] = dg, db
    assert abs(v - want_e) <= 1e-10 * max(1.0, abs(want_e))
    assert rel_err(g, want) <= 1e-10
    assert rel_err(psi, want_psi) <= 1e-10


@pytest.mark.parametrize("fam", ["5", "6", "r2m3", "pair"])
@pytest.mark.parametrize("n,p", [(21, 2), (27, 2), (30, 2)])
def test_chain_register_families(n, p, fam, monkeypatch):
    """single-vector sweeps with 32 amplitudes per thread (R=5: B windows need one
    exchange per pass; family 6 = two independent warp groups per CTA) against the
    default R=4 family"""
    env = {"r2m3": {"QSB_SWEEP_R2M": "3"}, "pair": {"QSB_PAIR": "2"}}.get(fam, {"QSB_SWEEP_R1M": fam, "QSB_SWEEP_R1": fam})
    if not variant_available(env):
        pytest.skip(f"{env}: an A/B experiment sweep family (build with tools/build_variant.py QSB_VARIANTS=1)")
    poly = random_instance(300 + n, n)
    params = params_wide(11 * n + p, p)
    ref = run(poly, params, monkeypatch, merge=True)
    if fam == "r2m3":  # merged bra/ket sweeps with 16 warps x 8 amplitudes per vector
        monkeypatch.setenv("QSB_SWEEP_R2M", "3")
    elif fam == "pair":  # single-vector B sweeps as lock-stepped 2-CTA clusters
        monkeypatch.setenv("QSB_PAIR", "2")
    else:
        monkeypatch.setenv("QSB_SWEEP_R1M", fam)
        monkeypatch.setenv("QSB_SWEEP_R1", fam)
    got = run(poly, params, monkeypatch, merge=True)
    assert abs(got[0] - ref[0]) <= 1e-12 * max(1.0, abs(ref[0]))
    assert rel_err(got[1], ref[1]) <= 1e-12
    assert rel_err(got[3], ref[3]) <= 1e-12


@pytest.mark.parametrize("n,p", [(16, 3), (30, 1)])
def test_gradient_without_value(n, p, monkeypatch):
    """gradient() asks for no <C>: the bridge sweep must still read the table (bra = C*ket)"""
    poly = random_instance(500 + n, n)
    params = params_wide(3 * n + p, p)
    h = qs.create_handle(poly, backend_name="b200")
    v, g = qs.value_and_grad(h, params)
    g2 = qs.gradient(h, params)
    h.close()
    assert rel_err(flat(g2), flat(g)) <= 1e-13


@pytest.mark.parametrize("n,p", [(3, 1), (6, 3), (9, 2), (11, 4)])
def test_small_register_kernel_is_bit_exact(n, p, monkeypatch):
    """n <= 11: the whole circuit runs in one CTA with the reference's arithmetic
    (small.cu) -- <C>, gradient and final state equal the numba-order oracle bit for
    bit on integral tables, in fast and exact mode alike."""
    poly = random_instance(900 + n, n)
    params = params_wide(17 * n + p, p)
    table = oracle.precompute_table(poly.weights, poly.masks, n)
    want_psi = oracle.simulate(table, n, params.gammas, params.betas)
    want_e = oracle.expectation(table, want_psi)
    dg, db = oracle.gradient(table, want_psi.copy(), params.gammas, params.betas)
    for exact in ("0", "1"):
        monkeypatch.setenv("QAOA_B200_EXACT", exact)
        h = qs.create_handle(poly, backend_name="b200")
        v, g = qs.value_and_grad(h, params)
        psi = np.asarray(qs.statevector(h, params))
        h.close()
        assert v == min(max(want_e, table.min()), table.max())
        assert np.array_equal(np.array(g.d_gammas), dg) and np.array_equal(np.array(g.d_betas), db)
        assert np.array_equal(psi, want_psi)
