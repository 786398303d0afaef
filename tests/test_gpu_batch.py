"""Many-instance calls (paper_2407_13012_b200/batch.py) against the CPU oracle: the
one-CTA launch for n <= 11 and the concurrent-streams path (qsb_value_and_grad_many)
for 12 <= n <= 22, mixed in one call, in input order."""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import batch

from conftest import random_instance, random_params, rel_err
from oracle import oracle

pytestmark = pytest.mark.gpu


def test_mixed_batch_vs_oracle(monkeypatch):
    sizes = [8, 13, 16, 12, 20, 11, 22, 17, 14, 16]
    polys = [random_instance(400 + k, n) for k, n in enumerate(sizes)]
    params = [random_params(500 + k, 1 + k % 4) for k in range(len(sizes))]
    handles = [qs.create_handle(p, backend_name="b200") for p in polys]
    got = batch.value_and_grad_batch(handles, params, threads=3)
    for h, poly, prm, (v, g) in zip(handles, polys, params, got):
        table = oracle.precompute_table(poly.weights, poly.masks, poly.n)
        e, dg, db = oracle.value_and_grad(table, poly.n, prm.gammas, prm.betas)
        e = min(max(e, table.min()), table.max())
        assert abs(v - e) <= 1e-10 * max(1.0, abs(e)), (poly.n, v, e)
        assert rel_err(np.concatenate([g.d_gammas, g.d_betas]), np.concatenate([dg, db])) <= 1e-10
        assert g.layer_applications == 6 * prm.p + 1
        # the batch equals the one-by-one call exactly (same kernels, same reductions) when
        # that call also runs without forward checkpoints (which store true values every
        # sweep instead of carrying the gate scale: equal to rounding)
        v2, g2 = qs.value_and_grad(h, prm)
        assert abs(v2 - v) <= 1e-12 * max(1.0, abs(v))
        assert rel_err(np.concatenate([g2.d_gammas, g2.d_betas]), np.concatenate([g.d_gammas, g.d_betas])) <= 1e-12
        monkeypatch.setenv("QSB_NO_CKPT", "1")
        v1, g1 = qs.value_and_grad(h, prm)
        monkeypatch.delenv("QSB_NO_CKPT")
        assert v1 == v and g1 == g
    # the kets are |+> afterwards (reference gradient contract)
    h = handles[4]
    plus = np.full(1 << h.n, 1.0 / np.sqrt(float(1 << h.n)))
    batch.value_and_grad_batch([h], [params[4]])
    assert np.max(np.abs(np.asarray(h.state.data) - plus)) <= 1e-12
    for hh in handles:
        hh.close()


def test_same_handle_twice_in_one_batch(monkeypatch):
    """two instances on one context run one after the other (shared partials scratch)"""
    monkeypatch.setenv("QSB_NO_CKPT", "1")  # bitwise comparison with the one-by-one calls
    poly = random_instance(77, 15)
    h = qs.create_handle(poly, backend_name="b200")
    p1, p2 = random_params(1, 2), random_params(2, 3)
    (va, ga), (vb, gb) = batch.value_and_grad_batch([h, h], [p1, p2])
    assert (va, ga) == qs.value_and_grad(h, p1)
    assert (vb, gb) == qs.value_and_grad(h, p2)
    h.close()
