"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
It imports the reference package `qaoasim` from /root/reference/pkg/src and uses
its "accelerated" (numba) kernel set — the bitwise anchor named in SURVEY.md
§8(a) — plus its graph generators and seeds, and writes small .npz fixtures next
to this script.  Nothing at test time reads /root/reference.

Large vectors are stored as sha256 digests (little-endian raw bytes); vectors
up to 2^12 entries are stored in full.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["QAOA_KERNELS"] = "accelerated"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

import qaoasim as qs  # noqa: E402  (the reference)
from qaoasim import adjoint, backend, circuit, rng  # noqa: E402
from qaoasim.kernels import numba_impl  # noqa: E402

BACKEND = "accelerated"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_params(seed: int, p: int, scale: float = 2.0):
    # reference tests/conftest.py:59-63
    stream = rng.Stream(seed)
    betas = [(stream.next_uniform() - 0.5) * scale for _ in range(p)]
    gammas = [(stream.next_uniform() - 0.5) * scale for _ in range(p)]
    return qs.QaoaParams(betas=betas, gammas=gammas)


def qubo_polynomial(n: int, seed: int) -> qs.Polynomial:
    """Dense QUBO: n linear + n(n-1)/2 pair terms, weights (U-0.5)*8 (float)."""
    st = rng.Stream(seed)
    terms = [((st.next_uniform() - 0.5) * 8.0, 1 << i) for i in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            terms.append(((st.next_uniform() - 0.5) * 8.0, (1 << i) | (1 << j)))
    return qs.Polynomial(n, terms)


def weighted_maxcut(n: int, seed: int) -> qs.Polynomial:
    """Complete graph with integer weights 1 + floor(8U) (bit-exact integral table)."""
    st = rng.Stream(seed)
    edges = [(u, v, float(1 + int(8 * st.next_uniform()))) for u in range(n) for v in range(u + 1, n)]
    return qs.maxcut_polynomial(qs.Graph(n, edges))


def run_case(name: str, poly: qs.Polynomial, params: qs.QaoaParams, shots: int, seed: int, full: bool):
    h = qs.create_handle(poly, backend_name=BACKEND)
    table = np.array(h.table.values.data, copy=True)
    psi = qs.statevector(h, params)
    e = qs.expectation(h, params)
    rec = {
        "n": poly.n,
        "weights": np.asarray(poly.weights),
        "masks": np.asarray(poly.masks),
        "betas": np.asarray(params.betas),
        "gammas": np.asarray(params.gammas),
        "table_sha": sha(table),
        "state_sha": sha(psi),
        "table_min": h.table.min_value,
        "table_max": h.table.max_value,
        "expectation": e,
    }
    if params.p >= 1:
        g = qs.gradient(h, params)
        rec["d_gammas"] = np.asarray(g.d_gammas)
        rec["d_betas"] = np.asarray(g.d_betas)
    if shots:
        qs.simulate(h, params)
        ss = qs.draw(h, shots, seed)
        rec["shots"] = shots
        rec["seed"] = seed
        rec["sample_idx"] = np.array([b for b, _ in ss.records], dtype=np.int64)
        rec["sample_cost"] = np.array([c for _, c in ss.records], dtype=np.float64)
    if full:
        rec["table"] = table
        rec["state"] = psi
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(f"{name}: n={poly.n} p={params.p} E={e!r}")


def kernel_kats():
    """Kernel-level vectors through the reference's own numba kernels."""
    r = np.random.default_rng(123)
    size = 1 << 11
    a = r.normal(size=size) + 1j * r.normal(size=size)
    a /= np.linalg.norm(a)
    b = r.normal(size=size) + 1j * r.normal(size=size)
    b /= np.linalg.norm(b)
    table = r.normal(size=size) * 3.0
    itable = np.floor(r.normal(size=size) * 5.0)
    out = {"a": a, "b": b, "table": table, "itable": itable}
    x = a.copy()
    numba_impl.phase_by_table(x, itable, 0.731)
    out["phase_itable"] = x
    x = a.copy()
    numba_impl.phase_by_table(x, table, 0.731)
    out["phase_table"] = x
    for j in (0, 1, 5, 10):
        x = a.copy()
        numba_impl.rx_qubit(x, j, 0.8, -0.6)
        out[f"rx_{j}"] = x
    x = a.copy()
    numba_impl.diag_scale(x, table)
    out["diag_scale"] = x
    w = np.empty(size)
    numba_impl.weighted_probs(a, table, w)
    out["weighted_probs"] = w
    out["tree_sum"] = np.array([numba_impl.tree_sum(w)])
    lengths = [1, 2, 7, 1024, 3000, 1 << 14, 100003]
    for L in lengths:
        v = np.random.default_rng(L).normal(size=L) * 100.0
        out[f"tree_in_{L}"] = v
        out[f"tree_out_{L}"] = np.array([numba_impl.tree_sum(v)])
    out["inner"] = np.array([numba_impl.inner(a, b)])
    out["diag_inner"] = np.array([numba_impl.diag_inner(a, table, b)])
    out["xsum"] = np.array([numba_impl.xsum(a, b, 11)])
    rr = np.random.default_rng(9)
    weights = rr.normal(size=40)
    masks = rr.integers(0, 1 << 10, size=40).astype(np.int64)
    pt = np.empty(1 << 10)
    numba_impl.precompute_table(weights, masks, pt)
    out["pre_weights"], out["pre_masks"], out["pre_table"] = weights, masks, pt
    # splitmix64 uniforms
    out["uniform_987"] = rng.uniform_block(987, 5, 100)
    out["uniform_big_seed"] = rng.uniform_block(2**63 + 11, 0, 64)
    # sampling from an uploaded state (point-mass-free, normalised)
    st = np.abs(r.normal(size=1 << 10)) + 0.01j
    st /= np.linalg.norm(st)
    ctx = backend.create_context(BACKEND)
    s = backend.alloc_plus_state(10, ctx)
    s.data[:] = st
    out["sample_state"] = st
    out["sample_idx_seed5"] = backend.sample_indices(s, 5000, seed=5)
    np.savez_compressed(OUT / "kernels.npz", **out)
    print("kernels.npz written")


def main():
    kernel_kats()
    # BASELINE.json config 1: MaxCut 3-regular n=16 p=3 ramp, 1024 shots seed 1
    g1 = qs.random_regular(16, 3, seed=1)
    run_case("c1_reg3_n16_p3", qs.maxcut_polynomial(g1), circuit.linear_ramp_params(3), 1024, 1, full=False)
    run_case("c1_reg3_n16_p3_random", qs.maxcut_polynomial(g1), random_params(7, 3), 1024, 9, full=False)
    # small cases with full vectors: MaxCut families, weighted, float QUBO
    cases = [
        ("k3_p1", qs.maxcut_polynomial(qs.Graph(3, [(0, 1), (1, 2), (0, 2)])), qs.QaoaParams([0.3], [0.4])),
        ("er8_p2", qs.maxcut_polynomial(qs.erdos_renyi(8, 0.5, seed=3)), random_params(11, 2)),
        ("reg3_n12_p4", qs.maxcut_polynomial(qs.random_regular(12, 3, seed=5)), random_params(12, 4)),
        ("wmaxcut_n12_p3", weighted_maxcut(12, 21), random_params(13, 3)),
        ("qubo_n12_p2", qubo_polynomial(12, 22), random_params(14, 2)),
        ("er13_p3", qs.maxcut_polynomial(qs.erdos_renyi(13, 0.4, seed=8)), random_params(15, 3)),
        ("reg3_n14_p2_ramp", qs.maxcut_polynomial(qs.random_regular(14, 3, seed=2)), circuit.linear_ramp_params(2)),
    ]
    for name, poly, params in cases:
        run_case(name, poly, params, 4096, 3, full=poly.n <= 12)
    # mid-size (hash + scalars only)
    run_case("qubo_n18_p2", qubo_polynomial(18, 31), random_params(16, 2), 2048, 4, full=False)
    run_case("wmaxcut_n20_p2", weighted_maxcut(20, 32), random_params(17, 2), 2048, 5, full=False)
    # BASELINE.json config 2: ER(24, 0.5) seed 1, p=4, ramp and random params
    g2 = qs.erdos_renyi(24, 0.5, seed=1)
    run_case("c2_er24_p4", qs.maxcut_polynomial(g2), circuit.linear_ramp_params(4), 0, 0, full=False)
    run_case("c2_er24_p4_random", qs.maxcut_polynomial(g2), random_params(1, 4), 0, 0, full=False)


if __name__ == "__main__":
    main()
