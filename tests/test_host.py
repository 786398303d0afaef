"""Host-side logic (no GPU): RNG, graph generators, polynomials, parameters,
the optimizer engine, the kernel registry and the public API surface.  Graph
and polynomial outputs are checked against the reference's golden inputs."""

import math

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import circuit, costpoly, kernels, optimizer, problems, rng
from paper_2407_13012_b200.errors import ContractViolation, ParseError

from conftest import brute_force_cut_table, golden, random_params


REFERENCE_ALL = [
    "BackendContext", "ContractViolation", "CostTable", "Gradient", "Graph", "OptimizeConfig", "OptimizeResult",
    "ParseError", "Polynomial", "QaoaParams", "RealBuffer", "ResourceError", "SampleSet", "SimHandle",
    "SpinPolynomial", "StateBuffer", "best_of", "complete_graph", "create_context", "create_handle", "cut_value",
    "draw", "erdos_renyi", "evaluate", "expectation", "generate_suite", "gradient", "histogram",
    "linear_ramp_params", "maxcut_polynomial", "minimize", "minimize_callback", "precompute", "random_regular",
    "read_graph", "read_terms", "sample", "simulate", "spin_to_boolean", "statevector", "write_graph",
    "write_terms", "__version__",
]


def test_public_api_is_a_superset_of_the_reference():
    for name in REFERENCE_ALL:
        assert name in qs.__all__ and hasattr(qs, name), name


class TestRng:
    def test_matches_sequential_splitmix64(self):
        mask = (1 << 64) - 1

        def seq(seed, count):
            out, state = [], seed
            for _ in range(count):
                state = (state + 0x9E3779B97F4A7C15) & mask
                z = state
                z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
                z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
                out.append(z ^ (z >> 31))
            return out

        for seed in (0, 1, 42, 2**63 + 11):
            assert [rng.value_at(seed, t) for t in range(8)] == seq(seed, 8)

    def test_vectorized_matches_scalar_and_golden(self):
        k = golden("kernels")
        block = rng.uniform_block(987, 5, 100)
        assert list(block) == [rng.uniform_at(987, 5 + t) for t in range(100)]
        assert np.array_equal(block, k["uniform_987"])
        assert np.array_equal(rng.uniform_block(2**63 + 11, 0, 64), k["uniform_big_seed"])


class TestProblems:
    @pytest.mark.parametrize("name", ["c1_reg3_n16_p3", "c2_er24_p4", "reg3_n12_p4", "er8_p2", "er13_p3"])
    def test_generators_reproduce_reference_instances(self, name):
        g = golden(name)
        graphs = {
            "c1_reg3_n16_p3": lambda: qs.random_regular(16, 3, seed=1),
            "c2_er24_p4": lambda: qs.erdos_renyi(24, 0.5, seed=1),
            "reg3_n12_p4": lambda: qs.random_regular(12, 3, seed=5),
            "er8_p2": lambda: qs.erdos_renyi(8, 0.5, seed=3),
            "er13_p3": lambda: qs.erdos_renyi(13, 0.4, seed=8),
        }
        poly = qs.maxcut_polynomial(graphs[name]())
        assert np.array_equal(poly.weights, g["weights"]) and np.array_equal(poly.masks, g["masks"])

    def test_baseline_configs(self):
        assert qs.random_regular(30, 3, seed=1).num_edges == 45
        assert qs.erdos_renyi(24, 0.5, seed=1).num_edges == 150
        assert qs.random_regular(34, 3, seed=1).num_edges == 51

    def test_regular_degrees(self):
        g = qs.random_regular(20, 3, seed=4)
        deg = np.zeros(20, int)
        for u, v, _ in g.edges:
            deg[u] += 1
            deg[v] += 1
        assert set(deg.tolist()) == {3}

    def test_suite_size(self):
        assert len(qs.generate_suite()) == 444

    def test_graph_validation(self):
        with pytest.raises(ContractViolation):
            qs.Graph(3, [(0, 0)])
        with pytest.raises(ContractViolation):
            qs.Graph(3, [(0, 1), (0, 1)])
        with pytest.raises(ContractViolation):
            qs.random_regular(5, 3, seed=1)

    def test_cut_and_polynomial_agree(self):
        g = qs.erdos_renyi(7, 0.5, seed=3)
        poly = qs.maxcut_polynomial(g)
        brute = brute_force_cut_table(g)
        for x in range(1 << 7):
            assert qs.evaluate(poly, x) == brute[x] == -qs.cut_value(g, x)

    def test_graph_file_round_trip(self, tmp_path):
        g = qs.random_regular(10, 3, seed=2)
        qs.write_graph(tmp_path / "g.txt", g)
        assert qs.read_graph(tmp_path / "g.txt") == g
        (tmp_path / "bad.txt").write_text("3 2\n0 1\n")
        with pytest.raises(ParseError):
            qs.read_graph(tmp_path / "bad.txt")


class TestPolynomial:
    def test_mask_range(self):
        with pytest.raises(ContractViolation):
            qs.Polynomial(2, [(1.0, 4)])

    def test_k3_evaluate(self, k3_poly):
        assert [qs.evaluate(k3_poly, x) for x in range(8)] == [0, -2, -2, -2, -2, -2, -2, 0]

    def test_spin_to_boolean_matches_spin_evaluation(self):
        sp = qs.SpinPolynomial(4, [(1.5, 0b0011), (-0.5, 0b1100), (2.0, 0b0101), (0.25, 0)])
        bp = qs.spin_to_boolean(sp)
        for x in range(16):
            spins = [1 - 2 * ((x >> i) & 1) for i in range(4)]
            want = sum(w * math.prod(spins[i] for i in range(4) if (m >> i) & 1) for w, m in sp.terms)
            assert qs.evaluate(bp, x) == pytest.approx(want, abs=1e-12)

    def test_terms_round_trip(self, tmp_path):
        poly = qs.Polynomial(5, [(0.1, 0b11), (-2.5, 0b10100), (1e-17, 0)])
        qs.write_terms(tmp_path / "t.txt", poly)
        assert qs.read_terms(tmp_path / "t.txt") == poly


class TestParams:
    def test_ramp(self):
        p = qs.linear_ramp_params(4)
        assert p.betas == (0.75, 0.5, 0.25, 0.0) and p.gammas == (0.25, 0.5, 0.75, 1.0)

    def test_flatten_round_trip(self):
        params = qs.QaoaParams(betas=[1.0, 2.0], gammas=[3.0, 4.0])
        flat = circuit.flatten_params(params)
        assert list(flat) == [3.0, 1.0, 4.0, 2.0]
        assert circuit.unflatten_params(flat) == params

    def test_errors(self):
        with pytest.raises(ContractViolation):
            qs.QaoaParams([0.1], [0.1, 0.2])
        with pytest.raises(ContractViolation):
            qs.linear_ramp_params(0)
        with pytest.raises(ContractViolation):
            circuit.unflatten_params([1.0, 2.0, 3.0])


class TestOptimizerEngine:
    def test_quadratic(self):
        A = np.diag([1.0, 10.0, 100.0])

        def provider(x):
            return 0.5 * x @ A @ x, A @ x

        res = qs.minimize_callback(provider, [1.0, 1.0, 1.0])
        assert res.converged and res.value < 1e-10

    def test_rosenbrock(self):
        def provider(x):
            f = (1 - x[0]) ** 2 + 100 * (x[1] - x[0] ** 2) ** 2
            g = np.array([-2 * (1 - x[0]) - 400 * x[0] * (x[1] - x[0] ** 2), 200 * (x[1] - x[0] ** 2)])
            return f, g

        res = qs.minimize_callback(provider, [-1.2, 1.0], qs.OptimizeConfig(max_iterations=200))
        assert res.converged and np.allclose(res.x, [1.0, 1.0], atol=1e-5)

    def test_config_validation(self):
        with pytest.raises(ContractViolation):
            qs.OptimizeConfig(c1=0.9, c2=0.1)
        with pytest.raises(ContractViolation):
            qs.OptimizeConfig(memory=0)

    def test_gradient_shape_checked(self):
        with pytest.raises(ContractViolation):
            qs.minimize_callback(lambda x: (0.0, np.zeros(3)), [1.0, 2.0])


class TestRegistry:
    def test_b200_and_alias(self):
        assert kernels.get("b200") is kernels.get("gpu")
        assert kernels.backend_name(kernels.get("b200")) == "b200"

    @pytest.mark.parametrize("name", ["cuda", "reference", "accelerated", "numba"])
    def test_cpu_sets_and_cuda_are_unknown(self, name):
        with pytest.raises(ValueError):
            kernels.get(name)

    def test_env_default(self, monkeypatch):
        monkeypatch.setenv("QAOA_KERNELS", "gpu")
        assert kernels.default_backend() == "b200"
        monkeypatch.setenv("QAOA_KERNELS", "bogus")
        with pytest.raises(ValueError):
            kernels.default_backend()


class TestCeilings:
    def test_ceiling_checks_precede_allocation(self, monkeypatch):
        from paper_2407_13012_b200 import backend

        monkeypatch.setenv("QAOA_MAX_QUBITS", "40")
        monkeypatch.setenv("QAOA_MEM_CEILING_BYTES", str(16 << 30))
        with pytest.raises(qs.ResourceError, match=str((1 << 31) * 16)):
            backend.check_state_alloc(31)
        monkeypatch.delenv("QAOA_MAX_QUBITS")
        with pytest.raises(ContractViolation):
            backend.check_state_alloc(31)
        with pytest.raises(ContractViolation):
            backend.check_state_alloc(0)
