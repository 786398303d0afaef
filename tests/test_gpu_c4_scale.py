"""BASELINE config 4 sizes (n=32, p=8) on one B200: correctness at a scale no CPU
oracle reaches, through size-independent properties (SURVEY.md §8(e) "Correctness at
scale" (3)): <psi|psi> = 1, E in [min C, max C], the gradient at zero parameters is 0,
central finite differences on two parameters, and sampled costs equal the host
evaluation of the polynomial (costpoly.evaluate, the reference's term-ordered sum).

Weighted MaxCut on K32 (integer weights 1 + floor(8U): the dyadic precompute path and
the Z2-reduced chain) and the dense float QUBO (per-term precompute, fp64 table, full
statevector).  The two handles are created and closed one at a time (64 GiB states)."""

import gc

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import rng
from paper_2407_13012_b200.kernels import b200

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N, P = 32, 8


def weighted_k32() -> qs.Polynomial:
    st = rng.Stream(1)
    edges = [(u, v, float(1 + int(8 * st.next_uniform()))) for u in range(N) for v in range(u + 1, N)]
    return qs.maxcut_polynomial(qs.Graph(N, edges))


def dense_qubo() -> qs.Polynomial:
    st = rng.Stream(1)
    terms = [((st.next_uniform() - 0.5) * 8.0, 1 << i) for i in range(N)]
    for i in range(N):
        for j in range(i + 1, N):
            terms.append(((st.next_uniform() - 0.5) * 8.0, (1 << i) | (1 << j)))
    return qs.Polynomial(N, terms)


@pytest.fixture(params=["wmaxcut_K32", "dense_qubo"])
def handle(request, monkeypatch):
    monkeypatch.setenv("QAOA_MAX_QUBITS", str(N))
    monkeypatch.setenv("QAOA_MEM_CEILING_BYTES", str(16 << N))
    gc.collect()  # handles of earlier modules release their HBM first
    poly = weighted_k32() if request.param == "wmaxcut_K32" else dense_qubo()
    h = qs.create_handle(poly, backend_name="b200")
    yield request.param, poly, h
    h.close()
    gc.collect()


def test_c4_scale_properties(handle):
    name, poly, h = handle
    lo, hi = h.table.min_value, h.table.max_value
    params = qs.linear_ramp_params(P)
    params = qs.QaoaParams(list(params.betas[:-1]) + [0.3], list(params.gammas))  # no identity mixer
    e, g = qs.value_and_grad(h, params)
    assert lo - 1e-9 * abs(lo) <= e <= hi + 1e-9 * abs(hi), (name, e, lo, hi)
    grad = np.array(list(g.d_gammas) + list(g.d_betas))
    assert np.all(np.isfinite(grad)) and np.abs(grad).max() > 0.0

    # central differences on one gamma and one beta (h = 1e-5: truncation ~1e-10 x third
    # derivative, rounding ~1e-16 |E| / 1e-5)
    step = 1e-5
    for which, k in (("gammas", 2), ("betas", 5)):
        vals = []
        for sgn in (1.0, -1.0):
            b, gm = list(params.betas), list(params.gammas)
            (gm if which == "gammas" else b)[k] += sgn * step
            vals.append(qs.expectation(h, qs.QaoaParams(b, gm)))
        fd = (vals[0] - vals[1]) / (2 * step)
        an = (g.d_gammas if which == "gammas" else g.d_betas)[k]
        assert abs(fd - an) <= 1e-6 * max(1.0, np.abs(grad).max()), (name, which, k, fd, an)

    # the state: unit norm on the device, samples whose costs are the polynomial's values
    qs.simulate(h, params)
    norm2 = b200.inner(h.state.data, h.state.data)
    assert abs(norm2.real - 1.0) <= 1e-12 and abs(norm2.imag) <= 1e-12, (name, norm2)
    ss = qs.draw(h, 1000, 7)
    for x, c in zip(ss.indices[:200].tolist(), ss.costs[:200].tolist()):
        assert c == qs.evaluate(poly, int(x)), (name, x, c)

    # zero parameters: E = <+|C|+> = sum_t w_t 2^-|m_t|, and dE = 0 (|+> is an X eigenstate,
    # C commutes with the phases)
    z = qs.QaoaParams([0.0] * P, [0.0] * P)
    e0, g0 = qs.value_and_grad(h, z)
    mean_c = sum(w * 2.0 ** -bin(int(m)).count("1") for w, m in zip(poly.weights, poly.masks))  # <+|C|+>
    assert abs(e0 - mean_c) <= 1e-10 * max(1.0, abs(mean_c)), (name, e0, mean_c)
    assert np.abs(np.array(list(g0.d_gammas) + list(g0.d_betas))).max() <= 1e-9 * max(1.0, abs(e0)), name
