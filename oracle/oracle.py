"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle (qaoa_oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker or the timed CPU baseline; the product
package never does.  The oracle restates the reference's numba kernel set
(/root/reference/pkg/src/qaoasim/kernels/numba_impl.py) and orchestration
(circuit.py, adjoint.py, backend.py sampling) in C with FMA-free arithmetic and
glibc cos/sin; tests/test_oracle_golden.py pins it bit-for-bit against vectors
produced by the reference itself (tests/golden/).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_u64 = C.c_uint64
_lib = None


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "qaoa_oracle.cpp").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.or_tree_sum.restype = C.c_double
        L.or_expectation.restype = C.c_double
        L.or_reduce_min.restype = C.c_double
        L.or_reduce_max.restype = C.c_double
        L.or_sample.restype = C.c_int
        L.or_num_threads.restype = C.c_int
        for name in ("or_tree_sum", "or_reduce_min", "or_reduce_max"):
            getattr(L, name).argtypes = [_vp, _u64]
        L.or_expectation.argtypes = [_vp, _vp, C.c_int]
        L.or_sample.argtypes = [_vp, _vp, C.c_int, _u64, _u64, _vp, _vp, _dp]
        L.or_phase_by_table.argtypes = [_vp, _vp, _u64, C.c_double]
        L.or_rx_qubit.argtypes = [_vp, _u64, C.c_int, C.c_double, C.c_double]
        L.or_uniform.argtypes = [_u64, _u64, _u64, _vp]
        L.or_precompute_table.argtypes = [_vp, _vp, _u64, _vp, _u64]
        L.or_simulate.argtypes = [_vp, _vp, C.c_int, C.c_int, _vp, _vp]
        L.or_gradient.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp]
        L.or_inner.argtypes = [_vp, _vp, _u64, _vp]
        L.or_diag_inner.argtypes = [_vp, _vp, _vp, _u64, _vp]
        L.or_xsum.argtypes = [_vp, _vp, _u64, C.c_int, _vp]
        L.or_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return C.c_void_p(a.ctypes.data)


def num_threads() -> int:
    return lib().or_num_threads()


def set_num_threads(k: int) -> None:
    lib().or_set_num_threads(int(k))


def precompute_table(weights, masks, n: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = np.ascontiguousarray(masks, dtype=np.int64)
    out = np.empty(1 << n, dtype=np.float64)
    lib().or_precompute_table(_p(w), _p(m), _u64(w.shape[0]), _p(out), _u64(out.shape[0]))
    return out


def simulate(table: np.ndarray, n: int, gammas, betas) -> np.ndarray:
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().or_simulate(_p(table), _p(psi), C.c_int(n), C.c_int(g.shape[0]), _p(g), _p(b))
    return psi


def expectation(table: np.ndarray, psi: np.ndarray) -> float:
    n = psi.shape[0].bit_length() - 1
    return lib().or_expectation(_p(table), _p(psi), n)


def gradient(table: np.ndarray, psi: np.ndarray, gammas, betas):
    """Adjoint walk from the forward state psi (psi is consumed)."""
    n = psi.shape[0].bit_length() - 1
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    p = g.shape[0]
    bra = np.empty_like(psi)
    dg = np.empty(p)
    db = np.empty(p)
    lib().or_gradient(_p(table), _p(psi), _p(bra), C.c_int(n), C.c_int(p), _p(g), _p(b), _p(dg), _p(db))
    return dg, db


def value_and_grad(table: np.ndarray, n: int, gammas, betas):
    psi = simulate(table, n, gammas, betas)
    e = expectation(table, psi)
    dg, db = gradient(table, psi, gammas, betas)
    return e, dg, db


def sample(psi: np.ndarray, table: np.ndarray | None, shots: int, seed: int):
    n = psi.shape[0].bit_length() - 1
    idx = np.empty(shots, dtype=np.int64)
    cost = np.empty(shots, dtype=np.float64)
    total = C.c_double()
    rc = lib().or_sample(_p(psi), _p(table) if table is not None else None, n, shots, seed & ((1 << 64) - 1),
                         _p(idx), _p(cost) if table is not None else None, C.byref(total))
    if rc:
        raise ValueError(f"state is not normalized: sum of probabilities = {total.value!r}")
    return idx, (cost if table is not None else None)


def tree_sum(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().or_tree_sum(_p(v), v.shape[0])


def rx_qubit(psi: np.ndarray, j: int, c: float, s: float) -> None:
    lib().or_rx_qubit(_p(psi), psi.shape[0], j, c, s)


def phase_by_table(psi: np.ndarray, table: np.ndarray, gamma: float) -> None:
    lib().or_phase_by_table(_p(psi), _p(table), psi.shape[0], gamma)


def inner(a, b):
    out = np.empty(2)
    lib().or_inner(_p(a), _p(b), _u64(a.shape[0]), _p(out))
    return complex(out[0], out[1])


def diag_inner(a, t, b):
    out = np.empty(2)
    lib().or_diag_inner(_p(a), _p(t), _p(b), _u64(a.shape[0]), _p(out))
    return complex(out[0], out[1])


def xsum(a, b, nq):
    out = np.empty(2)
    lib().or_xsum(_p(a), _p(b), _u64(a.shape[0]), C.c_int(nq), _p(out))
    return complex(out[0], out[1])


def uniform(seed: int, start: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().or_uniform(seed & ((1 << 64) - 1), start, count, _p(out))
    return out
