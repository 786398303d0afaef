"""Correctness at scale for the sharded path on one B200 (a separate module so the
C3 fixture of test_gpu_large.py has released its 40 GiB first)."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_sharded_n31_matches_unsharded(monkeypatch):
    """Correctness at scale for the sharded path: a 31-qubit weighted
    MaxCut, p=2, random angles, on one B200 -- unsharded (32 GiB statevector) vs two
    virtual shards with the all-to-all qubit swap (the multi-GPU schedule); plus the
    size-independent checks (norm, E within [min, max], zero-parameter gradient 0,
    sharded samples = the gathered state's tree draw)."""
    from paper_2407_13012_b200 import dist, rng

    # per-position schedule (3 statevectors per shard); the window chain's fused swap
    # needs a 4th and does not fit next to two 2^30 shards x 2 table layouts (160+ GiB)
    monkeypatch.setenv("QSB_SHARD_CHAIN", "0")
    monkeypatch.setenv("QAOA_MAX_QUBITS", "31")
    monkeypatch.setenv("QAOA_MEM_CEILING_BYTES", str(40 << 30))
    n, p = 31, 2
    st = rng.Stream(31)
    g = qs.random_regular(n + 1, 3, seed=3)  # 32 vertices, keep the edges inside 0..30
    edges = [(u, v) for u, v, *_ in g.edges if u < n and v < n]
    poly = qs.Polynomial(n, [(w, m) for u, v in edges
                             for w, m in (((-1.0 - st.next_below(3)), 1 << u), (-1.0, 1 << v), (2.0, (1 << u) | (1 << v)))])
    params = qs.QaoaParams([0.61, -0.27], [0.33, 0.72])
    h = qs.create_handle(poly, backend_name="b200")
    v1, g1 = qs.value_and_grad(h, params)
    lo, hi = h.table.min_value, h.table.max_value
    h.close()
    del h
    sh = dist.ShardedHandle(poly, 1, dist.VirtualExchanger(1))
    v2, dg, db = sh.value_and_grad(params)
    assert abs(v2 - v1) <= 1e-11 * abs(v1)
    want = np.array(list(g1.d_gammas) + list(g1.d_betas))
    got = np.concatenate([dg, db])
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
    assert lo <= v2 <= hi
    _, zg, zb = sh.value_and_grad(qs.QaoaParams([0.0, 0.0], [0.0, 0.0]))
    assert np.max(np.abs(np.concatenate([zg, zb]))) < 1e-9
    sh.simulate(params)
    ss = sh.draw(100000, 5)
    for b, c in list(zip(ss.indices[:100].tolist(), ss.costs[:100].tolist())):
        assert c == qs.evaluate(poly, b)
    sh.close()


def test_sharded_chain_c3_golden():
    """C3 (MaxCut 3-regular n=30, p=6 ramp) on four virtual shards through the window
    chain with fused swap stores: the reference's golden <C> and gradient (BASELINE.md
    section 3) within 1e-10"""
    from paper_2407_13012_b200 import dist
    from test_gpu_large import C3_DB, C3_DG, C3_E

    poly = qs.maxcut_polynomial(qs.random_regular(30, 3, seed=1))
    sh = dist.ShardedHandle(poly, 2, dist.VirtualExchanger(2))
    v, dg, db = sh.value_and_grad(qs.linear_ramp_params(6))
    sh.close()
    assert abs(v - C3_E) <= 1e-10 * abs(C3_E)
    got = np.concatenate([dg, db])
    want = np.array(C3_DG + C3_DB)
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
