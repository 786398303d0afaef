"""Schedule variants of the window chain agree with the default schedule.

The sweep kernel has several selectable schedules (fused.cu `sweep_family`,
sweep_host.cu): the staggered bra/ket schedule (QSB_STAG / QSB_STAGP), the register
families per sweep kind (QSB_SWEEP_R1 / R1M / R2 / R2M), paired B sweeps (QSB_PAIR).
The defaults are the measured-fastest per window kind; every alternative is a correct
schedule of the same arithmetic and must give the same E, gradient and statevector to
fast-mode rounding (1e-12 relative; the reference's 1e-10 bar is checked against the
oracle in test_gpu_chain.py).  The variables are read at each launch, so they can be
switched inside one process.
"""

import numpy as np
import pytest

import paper_2407_13012_b200 as qs

from conftest import variant_available, random_instance, rel_err

pytestmark = pytest.mark.gpu

VARIANTS = [
    {"QSB_STAG": "0"},
    {"QSB_STAGP": "0"},
    {"QSB_STAGP": "3"},
    {"QSB_SWEEP_R2M": "3"},
    {"QSB_SWEEP_R2M": "4"},
    {"QSB_SWEEP_R2M": "3", "QSB_STAG": "0"},
    {"QSB_SWEEP_R1M": "4"},
    {"QSB_SWEEP_R1M": "5"},
    {"QSB_SWEEP_R1M": "6"},
    {"QSB_SWEEP_R1": "4"},
    {"QSB_SWEEP_R1": "5"},
    {"QSB_SWEEP_R1": "3"},
    {"QSB_SWEEP_R2": "3"},
    {"QSB_PAIR": "0"},
    {"QSB_PAIR": "3"},
    {"QSB_NO_MERGE": "1"},
]


def flat(g):
    out = np.empty(2 * g.p)
    out[0::2] = g.d_gammas
    out[1::2] = g.d_betas
    return out


def evaluate(h, params):
    v, g = qs.value_and_grad(h, params)
    psi = np.asarray(qs.statevector(h, params))
    return v, flat(g), psi


@pytest.mark.parametrize("n,p", [(21, 3), (24, 2), (26, 3)])
def test_schedule_variants_agree(n, p, monkeypatch):
    poly = random_instance(7000 + n, n)
    rs = np.random.default_rng(n + p)
    # wide angles: both factored gate forms occur
    params = qs.QaoaParams(list(rs.uniform(-3.0, 3.0, p)), list(rs.uniform(-1.5, 1.5, p)))
    h = qs.create_handle(poly, backend_name="b200")
    try:
        v0, g0, psi0 = evaluate(h, params)
        for env in VARIANTS:
            if not variant_available(env):  # an A/B experiment family not in this build
                continue
            with monkeypatch.context() as m:
                for k, val in env.items():
                    m.setenv(k, val)
                v, g, psi = evaluate(h, params)
            assert abs(v - v0) <= 1e-12 * max(1.0, abs(v0)), env
            assert rel_err(g, g0) <= 1e-12, env
            assert rel_err(psi, psi0) <= 1e-12, env
    finally:
        h.close()
