"""Many problems per call (no reference counterpart: the reference runs handles one
at a time, cli.py `bench --jobs` only overlaps them with threads) -- the regime of the
paper's 444-graph benchmark suite (problems.generate_suite, n = 6..29) and of
optimizer restarts.

* n <= 11: the whole circuit fits one CTA (small.cu); one launch runs one CTA per
  (handle, parameters) instance.  Bit-identical to the one-by-one calls.
* n >= 12 (value_and_grad): qsb_value_and_grad_many issues every instance's window
  chain on its handle's own CUDA stream before awaiting any, from a few host threads,
  so instances whose sweeps cover only 2^(n-12) tiles (a few SMs each at n <= 22) run
  concurrently instead of back to back.  Identical to the one-by-one calls (same
  kernels, same reductions).
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
    for h in handles:  # their buffers were last touched on their own streams
        h.ctx.synchronize()
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


def _run_many(handles, params_list, threads: int):
    """value_and_grad of n >= 12 instances through qsb_value_and_grad_many (see the
    module doc); returns [(value, d_gammas, d_betas)] in input order"""
    import threading

    count = len(handles)
    res: list = [None] * count
    # instances that share a context (the same handle twice) must be issued by one
    # thread: its partials scratch serves one walk at a time (the C call serialises them)
    slot: dict = {}
    chunks: list = [[] for _ in range(max(1, min(threads, count)))]
    for i, h in enumerate(handles):
        key = h.ctx.device.handle.value
        if key not in slot:
            slot[key] = len(slot) % len(chunks)
        chunks[slot[key]].append(i)
    chunks = [c for c in chunks if c]
    bras = []
    for h in handles:  # the adjoint buffer of each handle (allocated once, kept)
        bras.append(h._adjoint_state())
    errors: list = []

    def work(ids):
        try:
            ctxs = (C.c_void_p * len(ids))(*[handles[i].ctx.device.handle for i in ids])
            tabs = (C.c_void_p * len(ids))(*[b200.ensure_table_handle(handles[i].table.values.data,
                                                                     handles[i].n).ptr for i in ids])
            kets = (C.c_void_p * len(ids))(*[handles[i].state.overwrite_target().ptr for i in ids])
            brs = (C.c_void_p * len(ids))(*[bras[i].data.ptr for i in ids])
            ps = [params_list[i].p for i in ids]
            p_arr = (C.c_int * len(ids))(*ps)
            gam = np.ascontiguousarray(np.concatenate([np.asarray(params_list[i].gammas, np.float64) for i in ids]))
            bet = np.ascontiguousarray(np.concatenate([np.asarray(params_list[i].betas, np.float64) for i in ids]))
            out = np.empty(sum(1 + 2 * p for p in ps))
            call("qsb_value_and_grad_many", len(ids), ctxs, tabs, kets, brs, p_arr,
                 gam.ctypes.data_as(C.POINTER(C.c_double)), bet.ctypes.data_as(C.POINTER(C.c_double)),
                 out.ctypes.data_as(C.POINTER(C.c_double)))
            o = 0
            for i, p in zip(ids, ps):
                res[i] = (out[o], out[o + 1: o + 1 + p], out[o + 1 + p: o + 1 + 2 * p])
                o += 1 + 2 * p
        except Exception as exc:  # noqa: BLE001 -- re-raised on the calling thread
            errors.append(exc)

    workers = [threading.Thread(target=work, args=(ids,)) for ids in chunks[1:]]
    for w in workers:
        w.start()
    if chunks:
        work(chunks[0])
    for w in workers:
        w.join()
    for b in bras:
        b.free()
    if errors:
        raise errors[0]
    for h in handles:  # the walk leaves the ket at |+> by contract (adjoint.py:39-42)
        h.state.mark_plus()
    return res


def expectation_batch(handles, params_list) -> list[float]:
    """circuit.expectation for every (handle, params) pair, one launch."""
    return [circuit._clamp(h, float(v)) for h, (v, _, _) in zip(handles, _run(handles, params_list, 1))]


def value_and_grad_batch(handles, params_list, threads: int = 4) -> list[tuple[float, adjoint.Gradient]]:
    """adjoint.value_and_grad for every (handle, params) pair: n <= 11 instances in one
    launch, n >= 12 instances concurrently on their own streams (`threads` host
    threads issue them); results in input order.  Exact mode (QAOA_B200_EXACT=1) runs
    the n >= 12 instances one by one (the reference-order walk)."""
    from . import backend

    if len(handles) != len(params_list):
        raise ContractViolation("handles and params_list must have the same length")
    for prm in params_list:
        if prm.p < 1:
            raise ContractViolation("batched calls need depth p >= 1")
    small = [i for i, h in enumerate(handles) if h.n <= 11]
    mid = [i for i, h in enumerate(handles) if h.n > 11]
    raw: list = [None] * len(handles)
    if small:
        for i, r in zip(small, _run([handles[i] for i in small], [params_list[i] for i in small], 2)):
            raw[i] = r
    if mid:
        if backend.exact_mode():
            for i in mid:
                v, g = adjoint.value_and_grad(handles[i], params_list[i])
                raw[i] = (v, np.array(g.d_gammas), np.array(g.d_betas))
        else:
            for i, r in zip(mid, _run_many([handles[i] for i in mid], [params_list[i] for i in mid], threads)):
                raw[i] = r
    out = []
    for h, (v, dg, db) in zip(handles, raw):
        g = adjoint.Gradient(d_betas=tuple(float(x) for x in db), d_gammas=tuple(float(x) for x in dg),
                             layer_applications=adjoint.LAYER_APPLICATIONS_PER_DEPTH * len(dg)
                             + adjoint.LAYER_APPLICATIONS_CONSTANT)
        out.append((circuit._clamp(h, float(v)), g))
    return out
