"""`qaoasim.oracle` for the reference's tests (tests/ref/conftest.py): a brute-force
dense simulation that shares no code with the B200 path -- phases from per-entry
polynomial evaluation (costpoly.evaluate), the mixer as an explicit 2x2 matrix per
qubit, a sequential expectation, central finite differences.  Restates the
reference's qaoasim/oracle.py interface (dense_simulate, dense_expectation,
fd_gradient; n <= 14, step h > 0).  Test infrastructure only."""

from __future__ import annotations

import numpy as np

from paper_2407_13012_b200.circuit import QaoaParams
from paper_2407_13012_b200.costpoly import Polynomial, evaluate
from paper_2407_13012_b200.errors import ContractViolation

MAX_ORACLE_QUBITS = 14
DEFAULT_FD_STEP = 1e-5


def _values(poly: Polynomial) -> np.ndarray:
    if poly.n > MAX_ORACLE_QUBITS:
        raise ContractViolation(f"dense oracle is capped at n <= {MAX_ORACLE_QUBITS}, got {poly.n}")
    return np.array([evaluate(poly, x) for x in range(1 << poly.n)], dtype=np.float64)


def _circuit(values: np.ndarray, params: QaoaParams) -> np.ndarray:
    size = values.shape[0]
    n = size.bit_length() - 1
    psi = np.full(size, 1.0 / np.sqrt(size), dtype=np.complex128)
    for gamma, beta in zip(params.gammas, params.betas):
        psi = psi * np.exp(-1j * gamma * values)
        c, s = np.cos(-beta), np.sin(-beta)  # Rx(-2 beta): [[c, -i s], [-i s, c]]
        for j in range(n):
            v = psi.reshape(-1, 2, 1 << j)
            lo, hi = v[:, 0, :].copy(), v[:, 1, :].copy()
            v[:, 0, :] = c * lo - 1j * s * hi
            v[:, 1, :] = -1j * s * lo + c * hi
    return psi


def _expect(values: np.ndarray, psi: np.ndarray) -> float:
    total = 0.0
    for f, a in zip(values.tolist(), psi.tolist()):
        total += f * (a.real * a.real + a.imag * a.imag)
    return total


def dense_simulate(poly: Polynomial, params: QaoaParams) -> np.ndarray:
    return _circuit(_values(poly), params)


def dense_expectation(poly: Polynomial, params: QaoaParams) -> float:
    values = _values(poly)
    return _expect(values, _circuit(values, params))


def fd_gradient(poly: Polynomial, params: QaoaParams, h: float = DEFAULT_FD_STEP) -> np.ndarray:
    """central differences in [gamma_1, beta_1, ...] order"""
    values = _values(poly)
    if h <= 0.0:
        raise ContractViolation(f"finite-difference step must be > 0, got {h}")
    x0 = np.empty(2 * params.p)
    x0[0::2], x0[1::2] = params.gammas, params.betas
    out = np.empty_like(x0)
    for i in range(x0.shape[0]):
        e = np.zeros_like(x0)
        e[i] = h
        fp, fm = (_expect(values, _circuit(values, QaoaParams(betas=x[1::2], gammas=x[0::2])))
                  for x in (x0 + e, x0 - e))
        out[i] = (fp - fm) / (2.0 * h)
    return out
