"""Adjoint-mode gradient over all 2p angles (reference: adjoint.py:1-77).

Exactly two statevectors are live: the ket (the handle's own buffer) and a bra.
The whole walk is one device call (qsb_value_and_grad):
  forward  — p fused layers on the ket, <C> taken from the last sweep;
  backward — for i = p..1 the pair (bra, ket) is swept together: the first sweep
             of a layer builds bra = C*ket (i = p) or closes layer i+1
             (<bra|C|ket> -> d_gamma_{i+1}, then the inverse phase on both),
             every sweep accumulates sum_j <bra|X_j|ket> (-> d_beta_i) for the
             qubits whose pairs sit in registers just before applying Rx(+2beta_i)
             to both, and the last sweep of layer 1 yields d_gamma_1 without
             storing anything.
X_j commutes with every Rx and the diagonal C with every phase, so those
contractions can be evaluated inside the sweeps that apply the inverses.
QAOA_B200_EXACT=1 runs the reference's op-by-op walk with bit-identical kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import backend, circuit
from .errors import ContractViolation

LAYER_APPLICATIONS_PER_DEPTH = 6
LAYER_APPLICATIONS_CONSTANT = 1


@dataclass(frozen=True)
class Gradient:
    d_betas: tuple[float, ...]
    d_gammas: tuple[float, ...]
    layer_applications: int

    @property
    def p(self) -> int:
        return len(self.d_betas)


def _walk(handle: circuit.SimHandle, params: circuit.QaoaParams, want_value: bool):
    p = params.p
    if p < 1:
        raise ContractViolation("gradient needs depth p >= 1")
    bra = handle._adjoint_state()
    try:
        value, dg, db = handle.ctx.kernels.value_and_grad(
            handle.state.overwrite_target(), bra.data, handle.table.values.data, handle.n, params.gammas, params.betas,
            exact=backend.exact_mode(), want_value=want_value,
        )
    finally:
        bra.free()
    if not backend.exact_mode() and handle.n >= 12:
        # the fused walk's last sweep only contracts: the ket is |+> by contract (the
        # reference's gradient leaves it there), written lazily on the next read
        handle.state.mark_plus()
    n = handle.n
    # reference-equivalent instrumentation: forward, bra prep, 4p inverse layers, reductions
    levels = backend._reduction_levels(1 << n)
    handle.ctx._count(1 + p * (1 + n) + 2 + p * (n * (levels + 1) + 2 * n + (levels + 1) + 2))
    grad = Gradient(
        d_betas=tuple(float(x) for x in db),
        d_gammas=tuple(float(x) for x in dg),
        layer_applications=LAYER_APPLICATIONS_PER_DEPTH * p + LAYER_APPLICATIONS_CONSTANT,
    )
    return value, grad


def gradient(handle: circuit.SimHandle, params: circuit.QaoaParams) -> Gradient:
    """d<C>/d beta_i and d<C>/d gamma_i for every layer."""
    return _walk(handle, params, False)[1]


def value_and_grad(handle: circuit.SimHandle, params: circuit.QaoaParams) -> tuple[float, Gradient]:
    """Expectation and gradient from ONE forward simulation (the optimizer's provider)."""
    value, grad = _walk(handle, params, True)
    return circuit._clamp(handle, value), grad
