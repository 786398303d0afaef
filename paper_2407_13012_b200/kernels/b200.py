"""The ``b200`` kernel set: the reference's 14 kernel functions
(qaoasim/kernels/numba_impl.py:40-260) on DeviceArrays, plus the allocation
hooks and the fused entry points (simulate / value_and_grad / sample) that the
circuit, adjoint and sampling modules call.  Every function is a thin ctypes
call into libqsb.so; there is no host fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from .. import _lib
from .._lib import DeviceArray, DeviceContext, call

NAME = "b200"

_u64 = C.c_uint64


def _device_index() -> int:
    for var in ("QAOA_DEVICE", "LOCAL_RANK"):
        raw = os.environ.get(var)
        if raw:
            return int(raw)
    return 0


def open_device(device: int | None = None) -> DeviceContext:
    return DeviceContext(_device_index() if device is None else int(device))


def empty(dctx: DeviceContext, length: int, dtype) -> DeviceArray:
    return DeviceArray(dctx, length, dtype)


def copy_device(dst: DeviceArray, src: DeviceArray) -> None:
    call("qsb_d2d", dst.dctx.handle, dst.ptr, src.ptr, src.nbytes)


def _h(a: DeviceArray):
    return a.dctx.handle


def _out2():
    return (C.c_double * 2)()


# ------------------------------------------------------------------ the kernel set
def fill_plus(amps: DeviceArray) -> None:
    call("qsb_fill_plus", _h(amps), amps.ptr, len(amps))


def phase_by_table(amps: DeviceArray, table: DeviceArray, gamma: float) -> None:
    th = table.table
    if th is not None:
        call("qsb_table_phase", _h(amps), th.ptr, amps.ptr, float(gamma))
    else:
        call("qsb_phase_by_table", _h(amps), amps.ptr, table.ptr, len(amps), float(gamma))


def diag_scale(amps: DeviceArray, table: DeviceArray) -> None:
    call("qsb_diag_scale", _h(amps), amps.ptr, table.ptr, len(amps))


def rx_qubit(amps: DeviceArray, j: int, c: float, s: float) -> None:
    call("qsb_rx_qubit", _h(amps), amps.ptr, len(amps), int(j), float(c), float(s))


def rx_layer(amps: DeviceArray, n: int, theta: float, exact: bool = False) -> None:
    call("qsb_rx_layer", _h(amps), amps.ptr, int(n), float(theta), _lib.QSB_EXACT if exact else 0)


def weighted_probs(amps: DeviceArray, table: DeviceArray, out: DeviceArray) -> None:
    call("qsb_weighted_probs", _h(amps), amps.ptr, table.ptr, out.ptr, len(amps))


def probs(amps: DeviceArray, out: DeviceArray) -> None:
    call("qsb_probs", _h(amps), amps.ptr, out.ptr, len(amps))


def tree_sum(vals: DeviceArray) -> float:
    out = C.c_double()
    call("qsb_tree_sum", _h(vals), vals.ptr, len(vals), C.byref(out))
    return out.value


def reduce_min(vals: DeviceArray) -> float:
    out = C.c_double()
    call("qsb_reduce_min", _h(vals), vals.ptr, len(vals), C.byref(out))
    return out.value


def reduce_max(vals: DeviceArray) -> float:
    out = C.c_double()
    call("qsb_reduce_max", _h(vals), vals.ptr, len(vals), C.byref(out))
    return out.value


def inner(a: DeviceArray, b: DeviceArray) -> complex:
    out = _out2()
    call("qsb_inner", _h(a), a.ptr, b.ptr, len(a), out)
    return complex(out[0], out[1])


def diag_inner(a: DeviceArray, table: DeviceArray, b: DeviceArray) -> complex:
    out = _out2()
    call("qsb_diag_inner", _h(a), a.ptr, table.ptr, b.ptr, len(a), out)
    return complex(out[0], out[1])


def xsum(a: DeviceArray, b: DeviceArray, n_qubits: int) -> complex:
    out = _out2()
    call("qsb_xsum", _h(a), a.ptr, b.ptr, len(a), int(n_qubits), out)
    return complex(out[0], out[1])


def precompute_table(weights, masks, out: DeviceArray) -> None:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = np.ascontiguousarray(masks, dtype=np.int64)
    call("qsb_precompute_table", _h(out), w.ctypes.data, m.ctypes.data, w.shape[0], out.ptr, len(out))


def pairwise_level(src: DeviceArray, dst: DeviceArray) -> None:
    call("qsb_pairwise_level", _h(src), src.ptr, dst.ptr, len(dst))


# ------------------------------------------------------------------ cost-table object
class TableHandle:
    """Owns a qsb_table (compact index + LUT scratch) tied to a table DeviceArray."""

    def __init__(self, ptr: int, kind: int, nvals: int):
        self.ptr = ptr
        self.kind = kind
        self.nvals = nvals
        self._fin = weakref.finalize(self, _destroy_table, ptr)


def _destroy_table(ptr: int) -> None:
    lib = _lib._lib
    if lib is not None:
        lib.qsb_table_destroy(ptr)


def _attach(out: DeviceArray, ptr: C.c_void_p) -> None:
    kind, nvals = C.c_int(), C.c_int()
    call("qsb_table_kind", ptr, C.byref(kind), C.byref(nvals))
    out.table = TableHandle(ptr.value, kind.value, nvals.value)


def build_cost_table(n: int, weights, masks, out: DeviceArray) -> tuple[float, float]:
    """precompute_table + min/max + compact index in one call (qsb_table_create)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = np.ascontiguousarray(masks, dtype=np.int64)
    lo, hi, ptr = C.c_double(), C.c_double(), C.c_void_p()
    call(
        "qsb_table_create", _h(out), int(n), w.ctypes.data, m.ctypes.data, w.shape[0], out.ptr,
        C.byref(lo), C.byref(hi), C.byref(ptr),
    )
    _attach(out, ptr)
    return lo.value, hi.value


def ensure_table_handle(table: DeviceArray, n: int) -> TableHandle:
    """Attach a qsb_table to a user-filled table buffer (qsb_table_wrap)."""
    if table.table is None:
        ptr = C.c_void_p()
        call("qsb_table_wrap", _h(table), int(n), table.ptr, None, None, C.byref(ptr))
        _attach(table, ptr)
    return table.table


# ------------------------------------------------------------------ fused entry points
def _params(gammas, betas):
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    return g, b


def simulate(amps: DeviceArray, table: DeviceArray, n: int, gammas, betas, *, exact: bool, want_expectation: bool,
             half_ok: bool = False):
    """Reset to |+>, then p phase/mixer layers; optionally return <C> from the last sweep.

    half_ok: a Z2-reduced run (flip-symmetric table) may leave the upper half of amps
    unwritten -- returns (value, half) then, half = True when it did (mirror_state
    writes it)."""
    th = ensure_table_handle(table, n)
    g, b = _params(gammas, betas)
    flags = _lib.QSB_FROM_PLUS | (_lib.QSB_EXACT if exact else 0) | (_lib.QSB_HALF_OUT if half_ok else 0)
    e = C.c_double()
    call(
        "qsb_simulate_expect", _h(amps), th.ptr, amps.ptr, g.shape[0], _lib.f64_ptr(g), _lib.f64_ptr(b), flags,
        C.byref(e) if want_expectation else None,
    )
    value = e.value if want_expectation else None
    if not half_ok:
        return value
    half = C.c_int()
    call("qsb_ctx_last_half", _h(amps), C.byref(half))
    return value, bool(half.value)


def mirror_state(amps: DeviceArray, n: int) -> None:
    """psi(2^(n-1) + y) = psi(2^(n-1) - 1 - y): the upper half of a Z2-reduced state."""
    call("qsb_state_mirror", _h(amps), amps.ptr, int(n))


def table_symmetric(table: DeviceArray, n: int) -> bool:
    """the cost table is flip-symmetric bit for bit (C(x) = C(~x))"""
    th = ensure_table_handle(table, n)
    out = C.c_int()
    call("qsb_table_symmetric", th.ptr, C.byref(out))
    return bool(out.value)


def expectation(amps: DeviceArray, table: DeviceArray, n: int) -> float:
    th = ensure_table_handle(table, n)
    out = C.c_double()
    call("qsb_expectation", _h(amps), th.ptr, amps.ptr, 0, C.byref(out))
    return out.value


def value_and_grad(ket: DeviceArray, bra: DeviceArray, table: DeviceArray, n: int, gammas, betas, *, exact: bool,
                   skip_forward: bool = False, want_value: bool = True):
    th = ensure_table_handle(table, n)
    g, b = _params(gammas, betas)
    p = g.shape[0]
    dg = np.empty(p, dtype=np.float64)
    db = np.empty(p, dtype=np.float64)
    val = C.c_double()
    call(
        "qsb_value_and_grad", _h(ket), th.ptr, ket.ptr, bra.ptr, p, _lib.f64_ptr(g), _lib.f64_ptr(b),
        _lib.QSB_EXACT if exact else 0, 1 if skip_forward else 0, C.byref(val) if want_value else None,
        _lib.f64_ptr(dg), _lib.f64_ptr(db),
    )
    return (val.value if want_value else None), dg, db


def sample(amps: DeviceArray, table: DeviceArray | None, n: int, shots: int, seed: int, half: bool = False):
    """(indices int64[shots], costs f64[shots] or None).  half: amps holds only the lower
    half of a flip-symmetric state (qsb_sample_sym; same draws as the full state)."""
    th = ensure_table_handle(table, n).ptr if table is not None else None
    idx = np.empty(shots, dtype=np.int64)
    cost = np.empty(shots, dtype=np.float64) if table is not None else None
    total = C.c_double()
    call(
        "qsb_sample_sym" if half else "qsb_sample", _h(amps), th, amps.ptr, int(n), shots,
        int(seed) & ((1 << 64) - 1), idx.ctypes.data, cost.ctypes.data if cost is not None else None, C.byref(total),
    )
    return idx, cost
