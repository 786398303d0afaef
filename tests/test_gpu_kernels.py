"""Kernel-set parity on the B200: each of the 14 functions against vectors the
reference's numba kernels produced (tests/golden/kernels.npz) and against the
CPU oracle.  Bit-exact except phase_by_table on a non-integral table (device
sincos, <= 1e-15 as the reference's own cross-set tolerance)."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import backend as be
from paper_2407_13012_b200.errors import ContractViolation
from paper_2407_13012_b200.kernels import b200

from conftest import golden
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def k():
    return golden("kernels")


@pytest.fixture(scope="module")
def ctx():
    return be.create_context("b200")


def dev(ctx, values, dtype):
    values = np.asarray(values, dtype=dtype)
    d = b200.empty(ctx.device, values.shape[0], dtype)
    d[:] = values
    return d


def test_fill_plus(ctx):
    for n in (1, 2, 5, 13):
        d = b200.empty(ctx.device, 1 << n, np.complex128)
        b200.fill_plus(d)
        want = np.empty(1 << n, np.complex128)
        oracle.lib().or_fill_plus(oracle._p(want), oracle._u64(1 << n))
        assert np.array_equal(np.asarray(d), want)


def test_phase_integral_table_via_lut_bitwise(ctx, k):
    a = dev(ctx, k["a"], np.complex128)
    t = dev(ctx, k["itable"], np.float64)
    b200.ensure_table_handle(t, 11)
    assert t.table.kind == 1
    b200.phase_by_table(a, t, 0.731)
    assert np.array_equal(np.asarray(a), k["phase_itable"])


def test_phase_float_table_sincos(ctx, k):
    a = dev(ctx, k["a"], np.complex128)
    t = dev(ctx, k["table"], np.float64)
    b200.phase_by_table(a, t, 0.731)
    assert np.max(np.abs(np.asarray(a) - k["phase_table"])) < 1e-15


@pytest.mark.parametrize("j", [0, 1, 5, 10])
def test_rx_qubit_bitwise(ctx, k, j):
    a = dev(ctx, k["a"], np.complex128)
    b200.rx_qubit(a, j, 0.8, -0.6)
    assert np.array_equal(np.asarray(a), k[f"rx_{j}"])


def test_diag_scale_and_weighted_probs_bitwise(ctx, k):
    a = dev(ctx, k["a"], np.complex128)
    t = dev(ctx, k["table"], np.float64)
    out = b200.empty(ctx.device, len(a), np.float64)
    b200.weighted_probs(a, t, out)
    assert np.array_equal(np.asarray(out), k["weighted_probs"])
    assert b200.tree_sum(out) == float(k["tree_sum"][0])
    b200.diag_scale(a, t)
    assert np.array_equal(np.asarray(a), k["diag_scale"])


@pytest.mark.parametrize("length", [1, 2, 7, 1024, 3000, 1 << 14, 100003])
def test_tree_sum_bitwise(ctx, k, length):
    v = dev(ctx, k[f"tree_in_{length}"], np.float64)
    assert b200.tree_sum(v) == float(k[f"tree_out_{length}"][0])


def test_tree_sum_large_exact(ctx):
    v = dev(ctx, np.ones(1 << 20), np.float64)
    assert b200.tree_sum(v) == 1048576.0
    x = np.sin(np.arange(1 << 22) * 0.7) * 1e3
    assert b200.tree_sum(dev(ctx, x, np.float64)) == oracle.tree_sum(x)


def test_inner_products_bitwise(ctx, k):
    a = dev(ctx, k["a"], np.complex128)
    b = dev(ctx, k["b"], np.complex128)
    t = dev(ctx, k["table"], np.float64)
    assert b200.inner(a, b) == complex(k["inner"][0])
    assert b200.diag_inner(a, t, b) == complex(k["diag_inner"][0])
    assert b200.xsum(a, b, 11) == complex(k["xsum"][0])


def test_min_max(ctx, k):
    t = dev(ctx, k["table"], np.float64)
    assert b200.reduce_min(t) == k["table"].min()
    assert b200.reduce_max(t) == k["table"].max()


def test_precompute_bitwise(ctx, k):
    out = b200.empty(ctx.device, 1 << 10, np.float64)
    b200.precompute_table(k["pre_weights"], k["pre_masks"], out)
    assert np.array_equal(np.asarray(out), k["pre_table"])


@pytest.mark.parametrize("n,terms", [(20, 300), (23, 60), (7, 5)])
def test_precompute_random_polynomials_bitwise(ctx, n, terms):
    r = np.random.default_rng(n)
    w = r.normal(size=terms) * 3
    m = np.array([int(x) & int(y) for x, y in zip(r.integers(0, 1 << n, terms), r.integers(0, 1 << n, terms))],
                 dtype=np.int64)
    m[::7] = 0
    out = b200.empty(ctx.device, 1 << n, np.float64)
    lo, hi = b200.build_cost_table(n, w, m, out)
    want = oracle.precompute_table(w, m, n)
    assert np.array_equal(np.asarray(out), want)
    assert (lo, hi) == (want.min(), want.max())


@pytest.mark.parametrize("n,terms,shift,deg", [(12, 40, 0, 2), (13, 200, 0, 2), (16, 500, 3, 4), (20, 1500, 1, 2),
                                               (22, 90, 0, 6), (14, 0, 0, 2)])
def test_precompute_dyadic_bitwise(ctx, n, terms, shift, deg):
    """Dyadic weights (multiples of 2^-shift, negatives, any degree): the exact int64
    subset-sum path (table.cu k_precompute_zeta) equals the reference's term-ordered
    double sum bit for bit, and so does the per-term kernel (QSB_NO_ZETA=1)."""
    r = np.random.default_rng(100 + n)
    w = r.integers(-9, 10, terms).astype(np.float64) / (1 << shift)
    m = np.zeros(terms, dtype=np.int64)
    for k in range(terms):
        bits = r.choice(n, size=int(r.integers(0, deg + 1)), replace=False)
        m[k] = int(sum(1 << int(b) for b in bits))
    want = oracle.precompute_table(w, m, n)
    out = b200.empty(ctx.device, 1 << n, np.float64)
    lo, hi = b200.build_cost_table(n, w, m, out)
    assert np.array_equal(np.asarray(out), want)
    assert not np.signbit(np.asarray(out)[np.asarray(out) == 0]).any()  # +0.0 like the reference
    assert (lo, hi) == (want.min(), want.max())


@pytest.mark.parametrize("kind", ["maxcut", "weighted_maxcut", "spin_even", "spin_odd", "random"])
def test_dyadic_table_stats_match_device_passes(ctx, kind, monkeypatch):
    """The dyadic path's fused min/max and its host (term-algebra) flip-symmetry test
    give exactly what the device passes find on the table (QSB_NO_TABLE_STATS=1)."""
    n = 18
    r = np.random.default_rng(7)
    if kind == "maxcut":
        poly = qs.maxcut_polynomial(qs.erdos_renyi(n, 0.3, seed=5))
    elif kind == "weighted_maxcut":
        edges = [(u, v, float(r.integers(1, 9))) for u in range(n) for v in range(u + 1, n) if r.random() < 0.4]
        poly = qs.maxcut_polynomial(qs.Graph(n, edges))
    elif kind.startswith("spin"):  # spin monomials of even (symmetric) or mixed degree, expanded to boolean
        deg = [2, 4] if kind == "spin_even" else [1, 2, 3]
        terms = []
        for _ in range(40):
            bits = r.choice(n, size=int(r.choice(deg)), replace=False)
            terms.append((float(r.integers(-5, 6)), int(sum(1 << int(b) for b in bits))))
        poly = qs.spin_to_boolean(qs.SpinPolynomial(n, terms))
    else:
        w = r.integers(-9, 10, 60).astype(np.float64)
        m = np.array([int(r.integers(0, 1 << n)) & int(r.integers(0, 1 << n)) for _ in range(60)], dtype=np.int64)
        poly = qs.Polynomial(n, list(zip(w.tolist(), m.tolist())))
    out = b200.empty(ctx.device, 1 << n, np.float64)
    got = b200.build_cost_table(n, poly.weights, poly.masks, out) + (b200.table_symmetric(out, n),)
    monkeypatch.setenv("QSB_NO_TABLE_STATS", "1")
    out2 = b200.empty(ctx.device, 1 << n, np.float64)
    want = b200.build_cost_table(n, poly.weights, poly.masks, out2) + (b200.table_symmetric(out2, n),)
    t = np.asarray(out2)
    assert want == (t.min(), t.max(), bool(np.array_equal(t, t[::-1])))
    assert got == want
    if kind in ("maxcut", "weighted_maxcut", "spin_even"):
        assert got[2]


@pytest.mark.parametrize("n,terms", [(12, 7), (16, 5000), (21, 700)])
def test_precompute_float_tiled_bitwise(ctx, n, terms, monkeypatch):
    """Float weights (no regrouping allowed): the tiled kernel (terms compacted per 4096-x
    tile in order; > 2048 terms take several list passes) equals the oracle and the
    per-x kernel (QSB_NO_ZETA=2) bit for bit."""
    r = np.random.default_rng(300 + n)
    w = r.normal(size=terms) * 2.5
    m = np.array([int(x) & int(y) for x, y in zip(r.integers(0, 1 << n, terms), r.integers(0, 1 << n, terms))],
                 dtype=np.int64)
    m[::11] = 0
    want = oracle.precompute_table(w, m, n)
    out = b200.empty(ctx.device, 1 << n, np.float64)
    b200.build_cost_table(n, w, m, out)
    assert np.array_equal(np.asarray(out), want)
    monkeypatch.setenv("QSB_NO_ZETA", "2")
    out2 = b200.empty(ctx.device, 1 << n, np.float64)
    b200.build_cost_table(n, w, m, out2)
    assert np.array_equal(np.asarray(out2), want)


def test_precompute_dyadic_matches_per_term_kernel(ctx, monkeypatch):
    poly = qs.maxcut_polynomial(qs.erdos_renyi(21, 0.5, seed=3))
    a = b200.empty(ctx.device, 1 << 21, np.float64)
    b200.build_cost_table(21, poly.weights, poly.masks, a)
    monkeypatch.setenv("QSB_NO_ZETA", "1")
    b = b200.empty(ctx.device, 1 << 21, np.float64)
    b200.build_cost_table(21, poly.weights, poly.masks, b)
    assert np.array_equal(np.asarray(a), np.asarray(b))


def test_pairwise_level(ctx):
    x = np.random.default_rng(1).normal(size=4096)
    s = dev(ctx, x, np.float64)
    d = b200.empty(ctx.device, 2048, np.float64)
    b200.pairwise_level(s, d)
    assert np.array_equal(np.asarray(d), x[0::2] + x[1::2])


@pytest.mark.parametrize("n", [3, 11, 12, 13, 17, 21, 22])
def test_rx_layer_exact_is_bitwise(ctx, n):
    r = np.random.default_rng(n)
    psi = r.normal(size=1 << n) + 1j * r.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    d = dev(ctx, psi, np.complex128)
    b200.rx_layer(d, n, 0.917, exact=True)
    want = psi.copy()
    c, s = np.cos(0.917 / 2.0), np.sin(0.917 / 2.0)
    import math

    c, s = math.cos(0.917 / 2.0), math.sin(0.917 / 2.0)
    for j in range(n):
        oracle.rx_qubit(want, j, c, s)
    assert np.array_equal(np.asarray(d), want)


@pytest.mark.parametrize("n", [12, 13, 16, 21, 24])
@pytest.mark.parametrize("theta", [0.917, -2.5, 3.0])
def test_rx_layer_fast_within_tolerance(ctx, n, theta):
    r = np.random.default_rng(n)
    psi = r.normal(size=1 << n) + 1j * r.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    d = dev(ctx, psi, np.complex128)
    b200.rx_layer(d, n, theta, exact=False)
    want = psi.copy()
    import math

    c, s = math.cos(theta / 2.0), math.sin(theta / 2.0)
    for j in range(n):
        oracle.rx_qubit(want, j, c, s)
    got = np.asarray(d)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


def test_sampling_uploaded_state_bitwise(ctx, k):
    st = dev(ctx, k["sample_state"], np.complex128)
    idx, cost = b200.sample(st, None, 10, 5000, 5)
    assert cost is None
    assert np.array_equal(idx, k["sample_idx_seed5"])


@pytest.mark.parametrize("n", [1, 2, 11, 12, 20, 23])
def test_sampling_matches_oracle_bitwise(ctx, n):
    r = np.random.default_rng(100 + n)
    psi = r.normal(size=1 << n) + 1j * r.normal(size=1 << n)
    psi /= np.sqrt(oracle.tree_sum(np.abs(psi) ** 2))
    d = dev(ctx, psi, np.complex128)
    shots = 20000
    try:
        want, _ = oracle.sample(psi, None, shots, 77)
    except ValueError:
        pytest.skip("normalisation rounding")
    got, _ = b200.sample(d, None, n, shots, 77)
    assert np.array_equal(got, want)


def test_sampling_unnormalized_rejected(ctx):
    d = dev(ctx, [1.0, 1.0], np.complex128)
    with pytest.raises(ContractViolation, match="normalized"):
        b200.sample(d, None, 1, 10, 0)
