"""Pin the CPU oracle (oracle/qaoa_oracle.cpp) to vectors produced by the
reference itself (tests/golden/make_golden.py -> numba "accelerated" set).
Everything here is bit-exact: the oracle restates the numba arithmetic."""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, golden, params_from, poly_from

from oracle import oracle


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "kernels")


def test_golden_cases_present():
    assert "c1_reg3_n16_p3" in CASES and "c2_er24_p4" in CASES


@pytest.mark.parametrize("name", [c for c in CASES if not c.startswith("c2_")])
def test_oracle_reproduces_reference_bitwise(name):
    g = golden(name)
    n = int(g["n"])
    table = oracle.precompute_table(g["weights"], g["masks"], n)
    assert sha(table) == str(g["table_sha"])
    assert table.min() == float(g["table_min"]) and table.max() == float(g["table_max"])
    psi = oracle.simulate(table, n, g["gammas"], g["betas"])
    assert sha(psi) == str(g["state_sha"])
    e = oracle.expectation(table, psi)
    e = min(max(e, table.min()), table.max())
    assert e == float(g["expectation"])
    if "shots" in g:
        idx, cost = oracle.sample(psi, table, int(g["shots"]), int(g["seed"]))
        assert np.array_equal(idx, g["sample_idx"])
        assert np.array_equal(cost, g["sample_cost"])
    if "d_gammas" in g:
        dg, db = oracle.gradient(table, psi.copy(), g["gammas"], g["betas"])
        assert np.array_equal(dg, g["d_gammas"]) and np.array_equal(db, g["d_betas"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_er24_p4", "c2_er24_p4_random"])
def test_oracle_reproduces_reference_c2(name):
    g = golden(name)
    n = int(g["n"])
    table = oracle.precompute_table(g["weights"], g["masks"], n)
    assert sha(table) == str(g["table_sha"])
    psi = oracle.simulate(table, n, g["gammas"], g["betas"])
    assert sha(psi) == str(g["state_sha"])
    assert oracle.expectation(table, psi) == float(g["expectation"])
    dg, db = oracle.gradient(table, psi, g["gammas"], g["betas"])
    assert np.array_equal(dg, g["d_gammas"]) and np.array_equal(db, g["d_betas"])


def test_c2_golden_matches_baseline_md():
    # BASELINE.md section 3 (numba, survey container)
    g = golden("c2_er24_p4")
    assert str(g["table_sha"]).startswith("5af15826fb6fd3b2")
    assert str(g["state_sha"]).startswith("d64856ef19a2fb61")
    assert float(g["expectation"]) == -64.06573702485557
    c1 = golden("c1_reg3_n16_p3")
    assert str(c1["table_sha"]).startswith("a40fd462569d4f0d")
    assert str(c1["state_sha"]).startswith("fd996249c4223ffe")
    assert float(c1["expectation"]) == -16.716866710582078
    assert sha(c1["sample_idx"]).startswith("91cdd0548b484a8a")


@pytest.fixture(scope="module")
def k():
    return golden("kernels")


class TestKernelKats:
    def test_phase_integral_table(self, k):
        x = k["a"].copy()
        oracle.phase_by_table(x, k["itable"], 0.731)
        assert np.array_equal(x, k["phase_itable"])

    def test_phase_float_table(self, k):
        x = k["a"].copy()
        oracle.phase_by_table(x, k["table"], 0.731)
        assert np.array_equal(x, k["phase_table"])

    @pytest.mark.parametrize("j", [0, 1, 5, 10])
    def test_rx_qubit(self, k, j):
        x = k["a"].copy()
        oracle.rx_qubit(x, j, 0.8, -0.6)
        assert np.array_equal(x, k[f"rx_{j}"])

    @pytest.mark.parametrize("length", [1, 2, 7, 1024, 3000, 1 << 14, 100003])
    def test_tree_sum(self, k, length):
        assert oracle.tree_sum(k[f"tree_in_{length}"]) == float(k[f"tree_out_{length}"][0])

    def test_inner_products(self, k):
        a, b, t = k["a"], k["b"], k["table"]
        assert oracle.inner(a, b) == complex(k["inner"][0])
        assert oracle.diag_inner(a, t, b) == complex(k["diag_inner"][0])
        assert oracle.xsum(a, b, 11) == complex(k["xsum"][0])

    def test_precompute(self, k):
        t = oracle.precompute_table(k["pre_weights"], k["pre_masks"], 10)
        assert np.array_equal(t, k["pre_table"])

    def test_uniforms(self, k):
        assert np.array_equal(oracle.uniform(987, 5, 100), k["uniform_987"])
        assert np.array_equal(oracle.uniform(2**63 + 11, 0, 64), k["uniform_big_seed"])

    def test_sampling_uploaded_state(self, k):
        idx, _ = oracle.sample(k["sample_state"], None, 5000, 5)
        assert np.array_equal(idx, k["sample_idx_seed5"])

    def test_unnormalized_rejected(self):
        with pytest.raises(ValueError, match="normalized"):
            oracle.sample(np.ones(4, dtype=np.complex128), None, 10, 0)
