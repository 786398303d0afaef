"""ctypes binding of libqsb.so (include/qsb.h) and the device-array type.

This is the only place Python touches the C ABI.  Status codes map onto the
reference's error convention (errors.py:4-19): QSB_ENOMEM -> ResourceError,
QSB_EINVAL -> ContractViolation, everything else -> RuntimeError.  There is no
CPU fallback: if the library or a B200 is missing, every device operation
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ContractViolation, ResourceError

# QSB_LIB: an experiment build of the same library (tools/build_variant.py)
_LIB_PATH = Path(os.environ["QSB_LIB"]) if os.environ.get("QSB_LIB") else Path(__file__).resolve().parent / "libqsb.so"

QSB_OK, QSB_EINVAL, QSB_ENOMEM, QSB_ECUDA, QSB_ENODEV = 0, 1, 2, 3, 4
QSB_EXACT = 1
QSB_FROM_PLUS = 2
QSB_HALF_OUT = 4

_vp = C.c_void_p
_u64 = C.c_uint64
_i32 = C.c_int
_dbl = C.c_double
_dp = C.POINTER(C.c_double)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "qsb_last_error": [],
    "qsb_abi_version": [],
    "qsb_has_variants": [],
    "qsb_device_count": [C.POINTER(_i32)],
    "qsb_ctx_create": [_i32, C.POINTER(_vp)],
    "qsb_ctx_destroy": [_vp],
    "qsb_ctx_sync": [_vp],
    "qsb_ctx_device": [_vp, C.POINTER(_i32)],
    "qsb_ctx_info": [_vp, C.POINTER(_i32), C.POINTER(_u64), C.POINTER(_u64)],
    "qsb_timer_start": [_vp],
    "qsb_timer_stop": [_vp, _dp],
    "qsb_ctx_launches": [_vp, C.POINTER(_u64)],
    "qsb_ctx_xfer": [_vp, C.POINTER(_u64), C.POINTER(_u64)],
    "qsb_prof_begin": [_vp],
    "qsb_prof_end": [_vp, _dp, _i32],
    "qsb_alloc": [_vp, _u64, C.POINTER(_vp)],
    "qsb_alloc_ipc": [_vp, _u64, C.POINTER(_vp)],
    "qsb_free": [_vp, _vp],
    "qsb_release_cached_memory": [_i32],
    "qsb_h2d": [_vp, _vp, _vp, _u64],
    "qsb_d2h": [_vp, _vp, _vp, _u64],
    "qsb_d2d": [_vp, _vp, _vp, _u64],
    "qsb_h2d_async": [_vp, _vp, _vp, _u64],
    "qsb_d2h_async": [_vp, _vp, _vp, _u64],
    "qsb_host_alloc": [_u64, C.POINTER(_vp)],
    "qsb_host_free": [_vp],
    "qsb_fill_plus": [_vp, _vp, _u64],
    "qsb_phase_by_table": [_vp, _vp, _vp, _u64, _dbl],
    "qsb_diag_scale": [_vp, _vp, _vp, _u64],
    "qsb_rx_qubit": [_vp, _vp, _u64, _i32, _dbl, _dbl],
    "qsb_weighted_probs": [_vp, _vp, _vp, _vp, _u64],
    "qsb_probs": [_vp, _vp, _vp, _u64],
    "qsb_tree_sum": [_vp, _vp, _u64, _dp],
    "qsb_reduce_min": [_vp, _vp, _u64, _dp],
    "qsb_reduce_max": [_vp, _vp, _u64, _dp],
    "qsb_inner": [_vp, _vp, _vp, _u64, _dp],
    "qsb_diag_inner": [_vp, _vp, _vp, _vp, _u64, _dp],
    "qsb_xsum": [_vp, _vp, _vp, _u64, _i32, _dp],
    "qsb_precompute_table": [_vp, _vp, _vp, _u64, _vp, _u64],
    "qsb_pairwise_level": [_vp, _vp, _vp, _u64],
    "qsb_table_create": [_vp, _i32, _vp, _vp, _u64, _vp, _dp, _dp, C.POINTER(_vp)],
    "qsb_table_wrap": [_vp, _i32, _vp, _dp, _dp, C.POINTER(_vp)],
    "qsb_table_create_mapped": [_vp, _i32, _i32, _vp, _vp, _u64, _i32, _i32, _i32, _u64, _vp, _dp, _dp,
                                C.POINTER(_vp)],
    "qsb_layer_sweeps": [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _dbl, C.c_uint, _dbl, _dp],
    "qsb_table_destroy": [_vp],
    "qsb_table_kind": [_vp, C.POINTER(_i32), C.POINTER(_i32)],
    "qsb_table_phase": [_vp, _vp, _vp, _dbl],
    "qsb_phase_lut_host": [_dbl, _dbl, _i32, _dp],
    "qsb_simulate": [_vp, _vp, _vp, _i32, _dp, _dp, C.c_uint],
    "qsb_simulate_expect": [_vp, _vp, _vp, _i32, _dp, _dp, C.c_uint, _dp],
    "qsb_rx_layer": [_vp, _vp, _i32, _dbl, C.c_uint],
    "qsb_expectation": [_vp, _vp, _vp, C.c_uint, _dp],
    "qsb_value_and_grad": [_vp, _vp, _vp, _vp, _i32, _dp, _dp, C.c_uint, _i32, _dp, _dp, _dp],
    "qsb_sample": [_vp, _vp, _vp, _i32, _u64, _u64, _vp, _vp, _dp],
    "qsb_sample_sym": [_vp, _vp, _vp, _i32, _u64, _u64, _vp, _vp, _dp],
    "qsb_sample_tree": [_vp, _vp, _i32, _dp],
    "qsb_shard_visit_run": [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _dp],
    "qsb_ipc_handle": [_vp, _vp, _vp],
    "qsb_ipc_open": [_vp, _vp, C.POINTER(_vp)],
    "qsb_ipc_close": [_vp, _vp],
    "qsb_device_sync": [_vp],
    "qsb_small_batch": [_vp, _i32, _vp, _vp, _vp, _dp, _dp, _i32, _dp],
    "qsb_sample_descend": [_vp, _vp, _vp, _i32, _u64, _vp, _vp, _vp],
    "qsb_scatter_chunks": [_vp, _vp, _u64, _i32, _vp, _u64],
    "qsb_value_and_grad_many": [_i32, _vp, _vp, _vp, _vp, _vp, _dp, _dp, _dp],
    "qsb_table_symmetric": [_vp, C.POINTER(_i32)],
    "qsb_state_mirror": [_vp, _vp, _i32],
    "qsb_ctx_last_half": [_vp, C.POINTER(_i32)],
    "qsb_fill_const": [_vp, _vp, _u64, _dbl, _dbl],
    "qsb_table_detach_values": [_vp],
    "qsb_nccl_version": [C.POINTER(_i32)],
    "qsb_nccl_unique_id": [_vp],
    "qsb_nccl_init": [_vp, _vp, _i32, _i32, C.POINTER(_vp)],
    "qsb_nccl_all_to_all": [_vp, _vp, _vp, _u64],
    "qsb_nccl_wait": [_vp, C.c_int64],
    "qsb_nccl_destroy": [_vp],
}
_RESTYPES = {"qsb_last_error": C.c_char_p, "qsb_abi_version": _i32, "qsb_has_variants": _i32}

# symbols declared in include/qsb.h (checked by the CPU test suite)
HEADER_SYMBOLS = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def library_path() -> Path:
    return _LIB_PATH


def load():
    """Load libqsb.so (building it first if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            from . import _build

            _build.build()
        lib = C.CDLL(str(_LIB_PATH))
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, _i32)
        _lib = lib
        return lib


def has_variants() -> bool:
    """the library carries the A/B experiment sweep families (tools/build_variant.py)"""
    return bool(load().qsb_has_variants())


def last_error() -> str:
    return load().qsb_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == QSB_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == QSB_EINVAL:
        raise ContractViolation(msg)
    if rc == QSB_ENOMEM:
        raise ResourceError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def dptr(x) -> C.c_double:
    return C.cast(x, _dp)


def f64_ptr(arr: np.ndarray):
    return arr.ctypes.data_as(_dp)


# ---------------------------------------------------------------- device context
class DeviceContext:
    """One B200 + one CUDA stream (qsb_ctx).  Fails loudly without a GPU."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _vp()
        check(lib.qsb_ctx_create(int(device), C.byref(h)), f"cannot open B200 device {device}")
        self.handle = h
        self.device = int(device)
        self._closed = False

    def sync(self) -> None:
        call("qsb_ctx_sync", self.handle)

    def info(self) -> tuple[int, int, int]:
        sms, free, total = _i32(), _u64(), _u64()
        call("qsb_ctx_info", self.handle, C.byref(sms), C.byref(free), C.byref(total))
        return sms.value, free.value, total.value

    def launches(self) -> int:
        out = _u64()
        call("qsb_ctx_launches", self.handle, C.byref(out))
        return out.value

    def xfer(self) -> tuple[int, int]:
        """(host->device, device->host) bytes copied by the library so far."""
        a, b = _u64(), _u64()
        call("qsb_ctx_xfer", self.handle, C.byref(a), C.byref(b))
        return a.value, b.value

    def prof_begin(self) -> None:
        call("qsb_prof_begin", self.handle)

    PROF_KINDS = 12

    @staticmethod
    def prof_kind_name(k: int) -> str:
        mode, nv, win = k // 4, (k // 2) % 2 + 1, "B" if k % 2 else "A"
        return f"{'single' if nv == 1 else 'braket'}{['', '_merged', '_bridge'][mode]}_{win}"

    def prof_end(self) -> dict:
        """{kind: (launches, total_ms, algorithmic_bytes)} per sweep kind, e.g.
        'single_A', 'braket_merged_B', 'braket_bridge_A' (kinds with no launch omitted)."""
        nk = self.PROF_KINDS
        out = (C.c_double * (3 * nk))()
        call("qsb_prof_end", self.handle, out, nk)
        return {self.prof_kind_name(k): (out[3 * k], out[3 * k + 1], out[3 * k + 2])
                for k in range(nk) if out[3 * k] > 0}

    def timer_start(self) -> None:
        call("qsb_timer_start", self.handle)

    def timer_stop(self) -> float:
        ms = _dbl()
        call("qsb_timer_stop", self.handle, C.byref(ms))
        return ms.value

    def close(self) -> None:
        if not self._closed and _lib is not None:
            self._closed = True
            _lib.qsb_ctx_destroy(self.handle)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceArray:
    """1-D array resident in B200 HBM.

    Behaves like the host ndarray the reference stores in StateBuffer.data /
    RealBuffer.data where the reference's tests touch it (backend.py:67-106):
    `buf[:] = values` uploads, `np.asarray(buf)` / `buf.copy()` / iteration /
    indexing download, `len()` and `==` work.  `free()` releases HBM eagerly.
    """

    __slots__ = ("dctx", "ptr", "dtype", "length", "table", "__weakref__")

    def __init__(self, dctx: DeviceContext, length: int, dtype, ipc: bool = False):
        """ipc=True: plain cudaMalloc memory that can be exported to peer processes
        (qsb_ipc_handle); otherwise buffers <= 1 GiB come from the stream-ordered pool."""
        self.dctx = dctx
        self.dtype = np.dtype(dtype)
        self.length = int(length)
        self.table = None  # attached qsb_table handle for cost tables
        p = _vp()
        fn = load().qsb_alloc_ipc if ipc else load().qsb_alloc
        check(fn(dctx.handle, self.nbytes, C.byref(p)), "device allocation")
        self.ptr = p.value

    # -- ndarray-like surface
    @property
    def nbytes(self) -> int:
        return self.length * self.dtype.itemsize

    @property
    def shape(self) -> tuple[int]:
        return (self.length,)

    @property
    def size(self) -> int:
        return self.length

    @property
    def ndim(self) -> int:
        return 1

    def __len__(self) -> int:
        return self.length

    def to_host(self, out: np.ndarray | None = None) -> np.ndarray:
        if self.ptr is None:
            raise ContractViolation("use of a freed device buffer")
        if out is None:
            out = np.empty(self.length, dtype=self.dtype)
        call("qsb_d2h", self.dctx.handle, out.ctypes.data, self.ptr, self.nbytes)
        return out

    def from_host(self, values) -> None:
        if self.ptr is None:
            raise ContractViolation("use of a freed device buffer")
        arr = np.ascontiguousarray(np.broadcast_to(np.asarray(values, dtype=self.dtype), (self.length,)))
        call("qsb_h2d", self.dctx.handle, self.ptr, arr.ctypes.data, self.nbytes)
        # a cost table written from the host: its cached compact index / LUT metadata
        # (qsb_table) is stale -- rebuilt from the new values on next use
        self.table = None

    def __array__(self, dtype=None, copy=None):
        host = self.to_host()
        return host if dtype is None else host.astype(dtype)

    def copy(self) -> np.ndarray:
        return self.to_host()

    def __iter__(self):
        return iter(self.to_host())

    def __getitem__(self, key):
        return self.to_host()[key]

    def __setitem__(self, key, value):
        if isinstance(key, slice) and key == slice(None):
            self.from_host(value)
            return
        host = self.to_host()
        host[key] = value
        self.from_host(host)

    def __eq__(self, other):
        if isinstance(other, (DeviceArray, np.ndarray, list, tuple, int, float, complex, np.generic)):
            return self.to_host() == np.asarray(other)
        return NotImplemented

    __hash__ = None

    # arithmetic on the host copy (the reference's tests combine table buffers with +,
    # e.g. test_costpoly.py:78-88); results are host ndarrays
    def _host(self, other):
        return other.to_host() if isinstance(other, DeviceArray) else other

    def __add__(self, o):
        return self.to_host() + self._host(o)

    def __radd__(self, o):
        return self._host(o) + self.to_host()

    def __sub__(self, o):
        return self.to_host() - self._host(o)

    def __rsub__(self, o):
        return self._host(o) - self.to_host()

    def __mul__(self, o):
        return self.to_host() * self._host(o)

    def __rmul__(self, o):
        return self._host(o) * self.to_host()

    def __truediv__(self, o):
        return self.to_host() / self._host(o)

    def __neg__(self):
        return -self.to_host()

    def __abs__(self):
        return np.abs(self.to_host())

    def __lt__(self, o):
        return self.to_host() < self._host(o)

    def __le__(self, o):
        return self.to_host() <= self._host(o)

    def __gt__(self, o):
        return self.to_host() > self._host(o)

    def __ge__(self, o):
        return self.to_host() >= self._host(o)

    @property
    def real(self) -> np.ndarray:
        return self.to_host().real

    @property
    def imag(self) -> np.ndarray:
        return self.to_host().imag

    def __repr__(self) -> str:
        return f"DeviceArray(len={self.length}, dtype={self.dtype}, device={self.dctx.device})"

    def free(self) -> None:
        if self.ptr is not None and _lib is not None:
            p, self.ptr = self.ptr, None
            # the context may already be gone (cyclic GC order): free without it
            _lib.qsb_free(None if self.dctx._closed else self.dctx.handle, p)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
