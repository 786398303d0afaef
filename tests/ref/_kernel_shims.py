"""Host-array kernel sets for the reference's tests/test_kernels_parity.py.

That file compares two kernel modules with numba_impl's signatures on host ndarrays
(qaoasim/kernels/numba_impl.py:40-260).  Under tests/ref/conftest.py:
  * `qaoasim.kernels.numpy_impl` -> ORACLE: the CPU oracle (oracle/qaoa_oracle.cpp,
    the bit-exact restatement of the numba set; test infrastructure);
  * `qaoasim.kernels.numba_impl` -> B200: every call uploads its arrays to HBM, runs
    the b200 kernel (libqsb.so), and copies the outputs back in place.
So the reference's parity tests check the B200 kernel set against the oracle.
"""

from __future__ import annotations

import ctypes as C
import types

import numpy as np

from oracle import oracle
from paper_2407_13012_b200 import _lib
from paper_2407_13012_b200.kernels import b200

_u64 = C.c_uint64


def _p(a):
    return C.c_void_p(np.ascontiguousarray(a).ctypes.data)


def make_oracle_set() -> types.ModuleType:
    L = oracle.lib()
    m = types.ModuleType("qaoasim.kernels.numpy_impl")
    m.NAME = "oracle"
    m.fill_plus = lambda amps: L.or_fill_plus(_p(amps), _u64(len(amps)))
    m.phase_by_table = lambda amps, table, gamma: oracle.phase_by_table(amps, np.ascontiguousarray(table), gamma)
    m.diag_scale = lambda amps, table: L.or_diag_scale(_p(amps), _p(np.ascontiguousarray(table)), _u64(len(amps)))
    m.rx_qubit = lambda amps, j, c, s: oracle.rx_qubit(amps, j, c, s)
    m.weighted_probs = lambda amps, table, out: L.or_weighted_probs(_p(amps), _p(table), _p(out), _u64(len(amps)))
    m.probs = lambda amps, out: L.or_probs(_p(amps), _p(out), _u64(len(amps)))
    m.tree_sum = lambda vals: oracle.tree_sum(vals)
    m.reduce_min = lambda vals: L.or_reduce_min(_p(np.ascontiguousarray(vals, dtype=np.float64)), len(vals))
    m.reduce_max = lambda vals: L.or_reduce_max(_p(np.ascontiguousarray(vals, dtype=np.float64)), len(vals))
    m.inner = lambda a, b: oracle.inner(a, b)
    m.diag_inner = lambda a, t, b: oracle.diag_inner(a, np.ascontiguousarray(t), b)
    m.xsum = lambda a, b, nq: oracle.xsum(a, b, nq)

    def precompute_table(weights, masks, out):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        mk = np.ascontiguousarray(masks, dtype=np.int64)
        L.or_precompute_table(_p(w), _p(mk), _u64(w.shape[0]), _p(out), _u64(out.shape[0]))

    m.precompute_table = precompute_table
    m.pairwise_level = lambda src, dst: L.or_pairwise_level(_p(src), _p(dst), _u64(len(dst)))
    return m


def make_b200_set() -> types.ModuleType:
    m = types.ModuleType("qaoasim.kernels.numba_impl")
    m.NAME = "b200"
    state = {}

    def dctx():
        if "d" not in state:
            state["d"] = b200.open_device()
        return state["d"]

    def up(a, dtype):
        d = _lib.DeviceArray(dctx(), len(a), dtype)
        d.from_host(np.asarray(a, dtype=dtype))
        return d

    def back(d, host):
        host[:] = d.to_host()
        d.free()

    def inplace(fn):
        def run(amps, *args):
            d = up(amps, np.complex128)
            dev_args = [up(x, np.float64) if isinstance(x, np.ndarray) else x for x in args]
            fn(d, *dev_args)
            back(d, amps)
            for x in dev_args:
                if isinstance(x, _lib.DeviceArray):
                    x.free()
        return run

    m.fill_plus = inplace(b200.fill_plus)
    m.phase_by_table = inplace(b200.phase_by_table)
    m.diag_scale = inplace(b200.diag_scale)
    m.rx_qubit = inplace(b200.rx_qubit)

    def weighted_probs(amps, table, out):
        a, t, o = up(amps, np.complex128), up(table, np.float64), up(out, np.float64)
        b200.weighted_probs(a, t, o)
        back(o, out)
        a.free(), t.free()

    def probs(amps, out):
        a, o = up(amps, np.complex128), up(out, np.float64)
        b200.probs(a, o)
        back(o, out)
        a.free()

    def scalar(fn, dtypes):
        def run(*args):
            devs = [up(x, dt) if dt is not None else x for x, dt in zip(args, dtypes)]
            try:
                return fn(*devs)
            finally:
                for x in devs:
                    if isinstance(x, _lib.DeviceArray):
                        x.free()
        return run

    c, f = np.complex128, np.float64
    m.weighted_probs = weighted_probs
    m.probs = probs
    m.tree_sum = scalar(b200.tree_sum, [f])
    m.reduce_min = scalar(b200.reduce_min, [f])
    m.reduce_max = scalar(b200.reduce_max, [f])
    m.inner = scalar(b200.inner, [c, c])
    m.diag_inner = scalar(b200.diag_inner, [c, f, c])
    m.xsum = scalar(b200.xsum, [c, c, None])

    def precompute_table(weights, masks, out):
        o = up(out, np.float64)
        b200.precompute_table(weights, masks, o)
        back(o, out)

    def pairwise_level(src, dst):
        s, d = up(src, np.float64), up(dst, np.float64)
        b200.pairwise_level(s, d)
        back(d, dst)
        s.free()

    m.precompute_table = precompute_table
    m.pairwise_level = pairwise_level
    return m
