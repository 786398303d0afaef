"""Kernel-set registry (the reference's plugin seam, kernels/__init__.py:13-65).

This package ships exactly one kernel set, ``b200`` (alias ``gpu``): hand-written
sm_100a CUDA behind the C ABI in include/qsb.h.  There is no CPU kernel set and
no fallback — the reference's ``reference``/``accelerated`` CPU sets are what
this replaces, and asking for them (or for ``cuda``) raises ValueError.
``QAOA_KERNELS`` selects the default (``b200``, ``gpu`` or ``auto``).
"""

import os

B200 = "b200"

_ALIASES = {"b200": B200, "gpu": B200}


def default_backend() -> str:
    choice = os.environ.get("QAOA_KERNELS", "auto").strip().lower()
    if choice == "auto":
        return B200
    if choice in _ALIASES:
        return _ALIASES[choice]
    raise ValueError(f"unknown QAOA_KERNELS value: {choice!r}")


def get(name: str | None = None):
    """Resolve a backend name to its kernel module."""
    if name is None:
        name = default_backend()
    resolved = _ALIASES.get(str(name).strip().lower())
    if resolved == B200:
        from . import b200

        return b200
    raise ValueError(f"unknown backend: {name!r} (available: b200, gpu)")


def backend_name(module) -> str:
    return getattr(module, "NAME", B200)
