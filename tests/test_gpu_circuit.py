"""End-to-end parity on the B200 through the public API (create_handle /
statevector / expectation / gradient / sample / minimize) against the golden
vectors the reference produced and the CPU oracle.

Bars (BASELINE.json north_star): cost tables bit-exact; samples bit-exact given
the same state and uniforms; statevector / expectation / gradient within 1e-10
relative (norm-wise).  In exact mode (QAOA_B200_EXACT=1) integral-table runs
must reproduce the reference bit for bit (statevector sha256)."""

import hashlib
import math

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import adjoint, backend as be, circuit
from paper_2407_13012_b200.errors import ContractViolation

from conftest import GOLDEN, golden, params_from, poly_from, random_instance, random_params, rel_err
from oracle import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "kernels")
INTEGRAL = [c for c in CASES if not c.startswith("qubo")]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(params=["fast", "exact"])
def mode(request, monkeypatch):
    monkeypatch.setenv("QAOA_B200_EXACT", "1" if request.param == "exact" else "0")
    return request.param


def flat_grad(g):
    out = np.empty(2 * g.p)
    out[0::2] = g.d_gammas
    out[1::2] = g.d_betas
    return out


@pytest.mark.parametrize("name", CASES)
def test_golden_case(name, mode):
    g = golden(name)
    poly, params = poly_from(g), params_from(g)
    h = qs.create_handle(poly, backend_name="b200")
    table = np.asarray(h.table.values.data)
    assert sha(table) == str(g["table_sha"])  # bit-exact for any weights
    assert (h.table.min_value, h.table.max_value) == (float(g["table_min"]), float(g["table_max"]))

    psi = qs.statevector(h, params)
    want_psi = oracle.simulate(table, poly.n, params.gammas, params.betas)
    assert sha(want_psi) == str(g["state_sha"])
    if mode == "exact" and name in INTEGRAL:
        assert sha(psi) == str(g["state_sha"])
    assert rel_err(psi, want_psi) <= TOL

    e = qs.expectation(h, params)
    assert abs(e - float(g["expectation"])) <= TOL * max(1.0, abs(float(g["expectation"])))
    if mode == "exact" and name in INTEGRAL:
        assert e == float(g["expectation"])

    grad = qs.gradient(h, params)
    want_g = np.empty(2 * params.p)
    want_g[0::2] = g["d_gammas"]
    want_g[1::2] = g["d_betas"]
    assert rel_err(flat_grad(grad), want_g) <= TOL
    if mode == "exact" and name in INTEGRAL:
        assert np.array_equal(flat_grad(grad), want_g)

    if "shots" in g:
        # samples are bit-exact given the same state and uniform draws
        qs.simulate(h, params)
        state_now = np.asarray(h.state.data)
        ss = qs.draw(h, int(g["shots"]), int(g["seed"]))
        want_idx, want_cost = oracle.sample(state_now, table, int(g["shots"]), int(g["seed"]))
        assert np.array_equal(ss.indices, want_idx) and np.array_equal(ss.costs, want_cost)
        if mode == "exact" and name in INTEGRAL:
            assert np.array_equal(ss.indices, g["sample_idx"])
        for b, c in ss.records[:50]:
            assert c == qs.evaluate(poly, b)


@pytest.mark.parametrize("seed", range(12))
def test_random_instances_vs_oracle(seed):
    n = 4 + seed * 2 % 19  # 4 .. 22
    p = 1 + seed % 5
    poly = random_instance(seed * 13 + 1, n)
    params = random_params(seed * 7 + 3, p)
    h = qs.create_handle(poly, backend_name="b200")
    table = np.asarray(h.table.values.data)
    v, grad = qs.value_and_grad(h, params)
    psi = oracle.simulate(table, n, params.gammas, params.betas)
    e = oracle.expectation(table, psi)
    dg, db = oracle.gradient(table, psi.copy(), params.gammas, params.betas)
    want = np.empty(2 * p)
    want[0::2], want[1::2] = dg, db
    assert abs(v - e) <= TOL * max(1.0, abs(e))
    assert rel_err(flat_grad(grad), want) <= TOL
    assert rel_err(qs.statevector(h, params), oracle.simulate(table, n, params.gammas, params.betas)) <= TOL


class TestReferenceBehaviour:
    """Ports of the reference's own unit tests (tests/test_circuit.py, test_adjoint.py,
    test_backend.py, test_sampling.py) against the b200 backend."""

    def test_triangle_table(self, k3_poly):
        h = qs.create_handle(k3_poly, backend_name="b200")
        assert list(h.table.values.data) == [0, -2, -2, -2, -2, -2, -2, 0]
        assert (h.table.min_value, h.table.max_value) == (-2.0, 0.0)

    def test_plus_states(self):
        ctx = be.create_context("b200")
        s = be.alloc_plus_state(1, ctx)
        assert s.data == pytest.approx([1 / math.sqrt(2)] * 2)
        assert list(be.alloc_plus_state(2, ctx).data) == [0.5 + 0j] * 4

    def test_phase_only_and_single_qubit_product(self):
        poly = qs.Polynomial(1, [(1.0, 0b1)])
        h = qs.create_handle(poly, backend_name="b200")
        qs.simulate(h, qs.QaoaParams([0.0], [math.pi]))
        assert h.state.data == pytest.approx([1 / math.sqrt(2), -1 / math.sqrt(2)], abs=1e-12)
        gamma, beta = math.pi / 2.0, math.pi / 8.0
        theta = -2.0 * beta
        rx = np.array([[math.cos(theta / 2), -1j * math.sin(theta / 2)],
                       [-1j * math.sin(theta / 2), math.cos(theta / 2)]])
        want = rx @ np.diag([1.0, np.exp(-1j * gamma)]) @ np.array([1, 1]) / math.sqrt(2)
        qs.simulate(h, qs.QaoaParams([beta], [gamma]))
        assert h.state.data == pytest.approx(want, abs=1e-12)

    def test_expectation_k3_and_p0_mean(self, k3_poly):
        h = qs.create_handle(k3_poly, backend_name="b200")
        assert qs.expectation(h, qs.QaoaParams([0.0], [0.0])) == pytest.approx(-1.5, abs=1e-12)
        poly = random_instance(17, 5)
        h = qs.create_handle(poly, backend_name="b200")
        assert qs.expectation(h, qs.QaoaParams((), ())) == pytest.approx(np.mean(h.table.values.data), abs=1e-12)

    def test_bounds(self):
        poly = random_instance(23, 14)
        h = qs.create_handle(poly, backend_name="b200")
        for seed in range(6):
            v = qs.expectation(h, random_params(seed, 3))
            assert h.table.min_value <= v <= h.table.max_value

    def test_zero_params_stationary(self):
        for seed, p, n in ((1, 1, 5), (2, 3, 13), (3, 6, 16)):
            h = qs.create_handle(random_instance(seed, n), backend_name="b200")
            g = qs.gradient(h, qs.QaoaParams([0.0] * p, [0.0] * p))
            assert np.max(np.abs(flat_grad(g))) <= 1e-12

    def test_exactly_two_statevectors_live(self, k3_poly):
        for poly in (k3_poly, random_instance(5, 14)):
            h = qs.create_handle(poly, backend_name="b200")
            h.ctx.reset_peak()
            qs.gradient(h, qs.linear_ramp_params(3))
            assert h.ctx.peak_live_statevectors == 2 and h.ctx.live_statevectors == 1

    def test_restoration(self):
        h = qs.create_handle(random_instance(77, 14), backend_name="b200")
        params = random_params(78, 4)
        before = qs.expectation(h, params)
        qs.gradient(h, params)
        assert qs.expectation(h, params) == pytest.approx(before, abs=1e-12)

    @pytest.mark.parametrize("n", [10, 14, 20])
    def test_state_after_gradient_is_plus(self, n):
        """adjoint.py:39-42: the gradient leaves the ket at |+>.  The fused walk (n >= 12)
        does not store its final uncompute -- the buffer is marked |+> and written on the
        first read, so reads and draws after gradient() / minimize() see |+>."""
        poly = random_instance(90 + n, n)
        h = qs.create_handle(poly, backend_name="b200")
        params = random_params(91, 3)
        qs.gradient(h, params)
        plus = np.full(1 << n, 1.0 / np.sqrt(float(1 << n)))
        assert np.max(np.abs(np.asarray(h.state.data) - plus)) <= 1e-12
        qs.value_and_grad(h, params)
        table = oracle.precompute_table(poly.weights, poly.masks, n)
        want_idx, want_cost = oracle.sample(plus.astype(np.complex128), table, 2000, 4)
        ss = qs.draw(h, 2000, 4)
        assert np.array_equal(ss.indices, want_idx) and np.array_equal(ss.costs, want_cost)
        qs.value_and_grad(h, params)
        mean = float(np.mean(table))
        assert circuit.expectation_of_state(h) == pytest.approx(mean, abs=1e-12 * max(1.0, abs(mean)))
        qs.simulate(h, params)  # a simulate after the pending fill is unaffected
        psi = oracle.simulate(table, n, params.gammas, params.betas)
        assert rel_err(np.asarray(h.state.data), psi) <= 1e-10

    def test_layer_applications(self, k3_poly):
        h = qs.create_handle(k3_poly, backend_name="b200")
        assert qs.gradient(h, qs.linear_ramp_params(2)).layer_applications == 13
        with pytest.raises(ContractViolation):
            qs.gradient(h, qs.QaoaParams((), ()))

    def test_reinitialises_between_calls(self):
        h = qs.create_handle(random_instance(3, 16), backend_name="b200")
        params = qs.linear_ramp_params(2)
        qs.simulate(h, params)
        first = h.state.data.copy()
        qs.simulate(h, params)
        assert np.array_equal(h.state.data.copy(), first)

    def test_sampling_determinism_and_costs(self):
        poly = random_instance(9, 13)
        h = qs.create_handle(poly, backend_name="b200")
        params = random_params(10, 2)
        a = qs.sample(h, params, 3000, seed=123)
        b = qs.sample(h, params, 3000, seed=123)
        assert a == b
        assert a.records != qs.sample(h, params, 3000, seed=124).records
        for bit, cost in a.records[:200]:
            assert cost == qs.evaluate(poly, bit)

    def test_sampling_fidelity(self):
        shots = 200_000
        poly = random_instance(33, 8)
        h = qs.create_handle(poly, backend_name="b200")
        params = random_params(34, 1)
        s = qs.sample(h, params, shots, seed=2024)
        probs = np.abs(qs.statevector(h, params)) ** 2
        counts = np.bincount(s.indices, minlength=probs.shape[0])
        assert 0.5 * np.sum(np.abs(counts / shots - probs)) < 0.02

    def test_sampling_errors(self):
        ctx = be.create_context("b200")
        st = be.alloc_plus_state(1, ctx)
        st.data[:] = [1.0, 1.0]
        with pytest.raises(ContractViolation, match="normalized"):
            be.sample_indices(st, 10, seed=0)
        with pytest.raises(ContractViolation):
            be.sample_indices(st, 0, seed=0)
        st.data[:] = [1.0] + [0.0]
        assert list(be.sample_indices(st, 100, seed=9)) == [0] * 100

    def test_backend_ops_and_counters(self):
        ctx = be.create_context("b200")
        state = be.alloc_plus_state(4, ctx)
        table = be.alloc_real(16, ctx)
        table.data[:] = np.arange(16.0)
        start = ctx.kernel_invocations
        be.apply_diagonal_phase(state, table, 0.7)
        be.apply_rx_layer(state, 0.9)
        out = be.export_state(state)
        assert np.sum(np.abs(out) ** 2) == pytest.approx(1.0, abs=1e-12)
        assert ctx.kernel_invocations > start
        clone = be.clone_state(state)
        assert ctx.live_statevectors == 2
        clone.free()
        clone.free()
        assert ctx.live_statevectors == 1
        want = sum(np.vdot(out, out[np.arange(16) ^ (1 << j)]) for j in range(4))
        assert be.xsum_inner(state, state) == pytest.approx(complex(want), abs=1e-12)

    def test_length_mismatch(self):
        ctx = be.create_context("b200")
        a = be.alloc_plus_state(1, ctx)
        b = be.alloc_plus_state(2, ctx)
        with pytest.raises(ContractViolation):
            be.inner_product(a, b)

    def test_optimizer_k3(self, k3_poly):
        h = qs.create_handle(k3_poly, backend_name="b200")
        res = qs.minimize(h, qs.linear_ramp_params(2))
        assert res.converged and res.value == pytest.approx(-2.0, abs=1e-6)


@pytest.mark.parametrize("name", ["c2_er24_p4", "c2_er24_p4_random"])
def test_c2_config(name, mode):
    """BASELINE config 2: ER(24, 0.5) p=4, gradient over all 8 parameters."""
    g = golden(name)
    poly, params = poly_from(g), params_from(g)
    h = qs.create_handle(poly, backend_name="b200")
    assert sha(np.asarray(h.table.values.data)) == str(g["table_sha"])
    v, grad = qs.value_and_grad(h, params)
    want = np.empty(8)
    want[0::2], want[1::2] = g["d_gammas"], g["d_betas"]
    assert abs(v - float(g["expectation"])) <= TOL * abs(float(g["expectation"]))
    assert rel_err(flat_grad(grad), want) <= TOL
    psi = qs.statevector(h, params)
    if mode == "exact":
        assert sha(psi) == str(g["state_sha"])
        assert np.array_equal(flat_grad(qs.gradient(h, params)), want)
