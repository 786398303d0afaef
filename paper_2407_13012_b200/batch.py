"""Many small problems in one device launch (no reference counterpart: the reference
runs handles one at a time, cli.py `bench --jobs` only overlaps them with threads).

For registers of n <= 11 qubits the whole circuit fits one CTA (small.cu); the batch
call puts one CTA per (handle, parameters) instance into a single launch -- the regime
of the paper's 444-graph benchmark suite (problems.generate_suite, n = 6..29) and of
optimizer restarts.  Results are bit-identical to the one-by-one calls.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import adjoint, circuit
from ._lib import call
from .errors import ContractViolation
from .kernels import b200


def _run(handles, params_list, mode: int):
    if len(handles) != len(params_list):
        raise ContractViolation("handles and params_list must have the same length")
    count = len(handles)
    if count == 0:
        return []
    dctx = handles[0].ctx.device
    tables, kets, ps = [], [], []
    for h, prm in zip(handles, params_list):
        if h.n > 11:
            raise ContractViolation(f"batched handles need n <= 11 qubits (got n={h.n}); call the handle directly")
        if prm.p < 1:
            raise ContractViolation("batched calls need depth p >= 1")
        if h.ctx.device.device != dctx.device:
            raise ContractViolation("batched handles must live on one device")
        tables.append(b200.ensure_table_handle(h.table.values.data, h.n).ptr)
        kets.append(h.state.data.ptr)
        ps.append(prm.p)
    gam = np.ascontiguousarray(np.concatenate([np.asarray(p.gammas, dtype=np.float64) for p in params_list]))
    bet = np.ascontiguousarray(np.concatenate([np.asarray(p.betas, dtype=np.float64) for p in params_list]))
    out = np.empty(sum(1 + 2 * p for p in ps), dtype=np.float64)
    t_arr = (C.c_void_p * count)(*tables)
    k_arr = (C.c_void_p * count)(*kets)
    p_arr = (C.c_int * count)(*ps)
    call("qsb_small_batch", dctx.handle, count, t_arr, k_arr, p_arr, gam.ctypes.data_as(C.POINTER(C.c_double)),
         bet.ctypes.data_as(C.POINTER(C.c_double)), mode, out.ctypes.data_as(C.POINTER(C.c_double)))
    res, o = [], 0
    for h, p in zip(handles, ps):
        res.append((out[o], out[o + 1: o + 1 + p], out[o + 1 + p: o + 1 + 2 * p]))
        o += 1 + 2 * p
    return res


def expectation_batch(handles, params_list) -> list[float]:
    """circuit.expectation for every (handle, params) pair, one launch."""
    return [circuit._clamp(h, float(v)) for h, (v, _, _) in zip(handles, _run(handles, params_list, 1))]


def value_and_grad_batch(handles, params_list) -> list[tuple[float, adjoint.Gradient]]:
    """adjoint.value_and_grad for every (handle, params) pair, one launch."""
    out = []
    for h, (v, dg, db) in zip(handles, _run(handles, params_list, 2)):
        g = adjoint.Gradient(d_betas=tuple(float(x) for x in db), d_gammas=tuple(float(x) for x in dg),
                             layer_applications=adjoint.LAYER_APPLICATIONS_PER_DEPTH * len(dg)
                             + adjoint.LAYER_APPLICATIONS_CONSTANT)
        out.append((circuit._clamp(h, float(v)), g))
    return out
