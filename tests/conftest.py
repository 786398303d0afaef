import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))

import paper_2407_13012_b200 as qs  # noqa: E402
from paper_2407_13012_b200 import rng  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (n >= 28)")


def _have_gpu() -> bool:
    try:
        import ctypes as C

        from paper_2407_13012_b200 import _lib

        n = C.c_int()
        return _lib.load().qsb_device_count(C.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


HAVE_GPU = _have_gpu()


# env knobs that select the A/B experiment sweep families, compiled only into a
# -DQSB_VARIANTS build (tools/build_variant.py); the product library omits them
_VARIANT_ONLY = {"QSB_STAG": {"0"}, "QSB_STAGP": {"0", "1", "2"}, "QSB_SWEEP_R1M": {"5"}, "QSB_SWEEP_R1MB": {"5"},
                 "QSB_SWEEP_R1": {"3", "5"}, "QSB_SWEEP_R2": {"3"}}


def variant_available(env: dict) -> bool:
    """True when the loaded library can run the sweep families `env` selects"""
    from paper_2407_13012_b200 import _lib

    if _lib.has_variants():
        return True
    return not any(env.get(k) in vals for k, vals in _VARIANT_ONLY.items())


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def poly_from(g: dict) -> qs.Polynomial:
    return qs.Polynomial(int(g["n"]), list(zip(g["weights"].tolist(), g["masks"].tolist())))


def params_from(g: dict) -> qs.QaoaParams:
    return qs.QaoaParams(betas=g["betas"], gammas=g["gammas"])


@pytest.fixture
def k3_poly():
    return qs.maxcut_polynomial(qs.Graph(3, [(0, 1), (1, 2), (0, 2)]))


# helpers mirroring the reference's tests/conftest.py:21-65 (same streams, same instances)
def brute_force_cut_table(g: qs.Graph) -> np.ndarray:
    table = np.zeros(1 << g.num_vertices)
    for x in range(1 << g.num_vertices):
        table[x] = -sum(w for u, v, w in g.edges if ((x >> u) ^ (x >> v)) & 1)
    return table


def random_polynomial(seed: int, n: int, max_terms: int = 50) -> qs.Polynomial:
    st = rng.Stream(seed)
    k = 1 + st.next_below(max_terms)
    terms = []
    for _ in range(k):
        mask = st.next_below(1 << n)
        terms.append(((st.next_uniform() - 0.5) * 8.0, mask))
    return qs.Polynomial(n, terms)


def random_instance(seed: int, n: int) -> qs.Polynomial:
    fams = ["er25", "er50", "er75", "complete"]
    if n >= 4 and n % 2 == 0:
        fams.append("reg3")
    st = rng.Stream(seed)
    fam = fams[st.next_below(len(fams))]
    if fam == "complete":
        g = qs.complete_graph(n)
    elif fam == "reg3":
        g = qs.random_regular(n, 3, st.derive(1))
    else:
        g = qs.erdos_renyi(n, {"er25": 0.25, "er50": 0.5, "er75": 0.75}[fam], st.derive(1))
    return qs.maxcut_polynomial(g)


def random_params(seed: int, p: int, scale: float = 2.0) -> qs.QaoaParams:
    st = rng.Stream(seed)
    betas = [(st.next_uniform() - 0.5) * scale for _ in range(p)]
    gammas = [(st.next_uniform() - 0.5) * scale for _ in range(p)]
    return qs.QaoaParams(betas=betas, gammas=gammas)


def rel_err(got, want) -> float:
    got = np.asarray(got)
    want = np.asarray(want)
    scale = max(float(np.max(np.abs(want))), 1e-300)
    return float(np.max(np.abs(got - want))) / scale
