"""Size-independent properties on the B200 path (the reference's property and
algorithm tests: norm preservation, central finite differences
of the expectation, bit-stable reductions, bounds)."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2407_13012_b200 as qs

from conftest import random_instance, random_params

pytestmark = pytest.mark.gpu


def flat(g):
    out = np.empty(2 * g.p)
    out[0::2] = g.d_gammas
    out[1::2] = g.d_betas
    return out


@pytest.mark.parametrize("n,p", [(9, 2), (13, 2), (17, 3), (21, 2)])
def test_gradient_matches_central_differences(n, p):
    """adjoint gradient (window chain / one-CTA kernel) vs central differences of
    expectation(); h = 1e-5 gives ~1e-9 absolute agreement (the reference's FD gate is
    rel 1e-5, test_adjoint.py:19-24)"""
    poly = random_instance(400 + n, n)
    rs = np.random.default_rng(n)
    betas, gammas = list(rs.uniform(-1, 1, p)), list(rs.uniform(-1, 1, p))
    h = qs.create_handle(poly, backend_name="b200")
    g = qs.gradient(h, qs.QaoaParams(betas, gammas))
    eps = 1e-5
    fd = []
    for i in range(p):  # flat order [g1, b1, g2, b2, ...]
        for which in ("g", "b"):
            def at(d):
                bb, gg = list(betas), list(gammas)
                (gg if which == "g" else bb)[i] += d
                return qs.expectation(h, qs.QaoaParams(bb, gg))
            fd.append((at(eps) - at(-eps)) / (2 * eps))
    h.close()
    fd = np.array(fd)
    assert np.max(np.abs(flat(g) - fd)) <= 1e-6 * max(1.0, np.max(np.abs(fd)))


@pytest.mark.parametrize("n", [11, 16, 24])
def test_reductions_are_bit_stable(n):
    """repeated calls give bit-identical <C> and gradients (fixed-order partial sums, no
    float atomics; test_backend.py:194-200)"""
    poly = random_instance(500 + n, n)
    params = qs.QaoaParams([0.3, -0.7], [0.9, 0.2])
    h = qs.create_handle(poly, backend_name="b200")
    runs = [qs.value_and_grad(h, params) for _ in range(3)]
    e = [qs.expectation(h, params) for _ in range(3)]
    h.close()
    assert runs[0][0] == runs[1][0] == runs[2][0]
    assert np.array_equal(flat(runs[0][1]), flat(runs[1][1])) and np.array_equal(flat(runs[1][1]), flat(runs[2][1]))
    assert e[0] == e[1] == e[2]


@settings(max_examples=12, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(n=st.integers(min_value=10, max_value=19), p=st.integers(min_value=1, max_value=3),
       seed=st.integers(min_value=0, max_value=10_000))
def test_norm_bounds_and_consistency(n, p, seed):
    poly = random_instance(seed, n)
    rs = np.random.default_rng(seed)
    params = qs.QaoaParams(list(rs.uniform(-3, 3, p)), list(rs.uniform(-2, 2, p)))
    h = qs.create_handle(poly, backend_name="b200")
    psi = np.asarray(qs.statevector(h, params))
    e = qs.expectation(h, params)
    v, _ = qs.value_and_grad(h, params)
    lo, hi = h.table.min_value, h.table.max_value
    h.close()
    assert abs(np.vdot(psi, psi).real - 1.0) <= 1e-12
    assert lo <= e <= hi
    assert abs(v - e) <= 1e-12 * max(1.0, abs(e))


def test_concurrent_handles_from_threads():
    """distinct handles may run concurrently (the reference's bench --jobs
    uses a thread pool): one CUDA stream per context, ctypes drops the GIL -- results
    equal the sequential ones bit for bit"""
    from concurrent.futures import ThreadPoolExecutor

    cases = [(random_instance(600 + k, n), n) for k, n in enumerate((9, 14, 17, 20, 12, 16))]
    params = qs.QaoaParams([0.4, -0.2], [0.7, 0.1])

    def run(case):
        poly, _ = case
        h = qs.create_handle(poly, backend_name="b200")
        out = [qs.value_and_grad(h, params) for _ in range(3)]
        h.close()
        return [(v, tuple(flat(g))) for v, g in out]

    seq = [run(c) for c in cases]
    with ThreadPoolExecutor(max_workers=6) as pool:
        par = list(pool.map(run, cases))
    assert par == seq


def test_batched_small_registers_equal_one_by_one():
    """batch.value_and_grad_batch: one CTA per instance in one launch (the paper's
    many-small-graphs regime) -- bit-identical to the per-handle calls"""
    from paper_2407_13012_b200 import batch

    suite = qs.generate_suite(vertex_range=(4, 11), instances=3, seed=7)
    handles, params = [], []
    rs = np.random.default_rng(1)
    for k, (_, graph) in enumerate(suite[:24]):  # (name, Graph) pairs, n = 4..11
        h = qs.create_handle(qs.maxcut_polynomial(graph), backend_name="b200")
        p = 1 + k % 4
        handles.append(h)
        params.append(qs.QaoaParams(list(rs.uniform(-1, 1, p)), list(rs.uniform(-1, 1, p))))
    got = batch.value_and_grad_batch(handles, params)
    eb = batch.expectation_batch(handles, params)
    for h, prm, (v, g), e in zip(handles, params, got, eb):
        v1, g1 = qs.value_and_grad(h, prm)
        assert v == v1 and e == v1
        assert g.d_gammas == g1.d_gammas and g.d_betas == g1.d_betas
        h.close()


def test_handles_reuse_large_blocks_bit_identically(monkeypatch):
    """Multi-GiB buffers (state, table, bra, forward checkpoints) go to the large-block
    cache on close and are reused by the next handle of the same size (ctx.cu): the
    results are bit-identical to runs without the cache (QSB_NO_BIGCACHE=1)."""
    params = random_params(5, 3)
    polys = [qs.maxcut_polynomial(qs.random_regular(27, 4, seed=s)) for s in (1, 2, 1)]
    got = []
    for poly in polys:
        h = qs.create_handle(poly, backend_name="b200")
        v, g = qs.value_and_grad(h, params)
        got.append((v, tuple(g.d_gammas), tuple(g.d_betas)))
        h.close()
    assert got[0] == got[2]
    monkeypatch.setenv("QSB_NO_BIGCACHE", "1")
    h = qs.create_handle(polys[1], backend_name="b200")
    v, g = qs.value_and_grad(h, params)
    h.close()
    assert got[1] == (v, tuple(g.d_gammas), tuple(g.d_betas))
    monkeypatch.delenv("QSB_NO_BIGCACHE")
    from paper_2407_13012_b200 import backend as be

    be.release_cached_memory()  # everything cached goes back; later handles allocate afresh
    h = qs.create_handle(polys[0], backend_name="b200")
    v, g = qs.value_and_grad(h, params)
    h.close()
    assert got[0] == (v, tuple(g.d_gammas), tuple(g.d_betas))
