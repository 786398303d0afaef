"""`import qaoasim` -> paper_2407_13012_b200 (the drop-in under the reference's own
tests; tests/ref/conftest.py puts this directory on sys.path and PYTHONPATH so that
subprocesses the tests spawn, e.g. `python -m qaoasim.cli`, see it too).

* every submodule the reference has resolves to this package's module of the same
  name (`qaoasim.oracle` -> tests/ref/_dense_oracle.py, the reference's brute-force
  test oracle restated; `qaoasim.kernels.numpy_impl` / `numba_impl` -> the CPU oracle /
  the b200 kernel set on host arrays, tests/ref/_kernel_shims.py);
* the reference's tests name its CPU kernel sets ("reference", "accelerated", "numpy",
  "numba") where any kernel set will do; under those tests the names resolve to
  "b200", the set that replaces them ("cuda" and other names still raise
  ValueError) -- per test in-process, via QSB_REF_ALIAS_NAMES=1 in subprocesses."""

import importlib
import sys
from pathlib import Path

_HERE = Path(__file__).resolve().parent
_REF = _HERE.parent.parent        # tests/ref
_ROOT = _REF.parent.parent        # repo root
for _p in (str(_ROOT), str(_REF)):
    if _p not in sys.path:
        sys.path.insert(0, _p)

import paper_2407_13012_b200 as _pkg  # noqa: E402
from paper_2407_13012_b200 import cli as _cli  # noqa: E402
from paper_2407_13012_b200 import kernels as _kernels  # noqa: E402

CPU_SET_NAMES = ("reference", "accelerated", "numpy", "numba")


def map_cpu_set_names() -> None:
    """resolve the reference's CPU kernel-set names to b200 (process-wide: used by
    subprocesses the reference's tests spawn; in-process tests/ref/conftest.py
    applies it per test with monkeypatch)"""
    for name in CPU_SET_NAMES:
        _kernels._ALIASES[name] = _kernels.B200
    _cli.BACKENDS = ("b200", "gpu", "reference", "accelerated")
    if "qaoasim.cli" in sys.modules:
        sys.modules["qaoasim.cli"].BACKENDS = _cli.BACKENDS


if __import__("os").environ.get("QSB_REF_ALIAS_NAMES") == "1":
    map_cpu_set_names()

# (cli is not pre-registered: `python -m qaoasim.cli` must load it through this
# package's path -- a second copy of paper_2407_13012_b200/cli.py named qaoasim.cli)
for _name in ("adjoint", "backend", "batch", "circuit", "costpoly", "errors", "kernels", "optimizer",
              "problems", "rng", "sampling"):
    sys.modules[f"qaoasim.{_name}"] = importlib.import_module(f"paper_2407_13012_b200.{_name}")

import _dense_oracle  # noqa: E402
from _kernel_shims import make_b200_set, make_oracle_set  # noqa: E402

_oracle_set, _b200_set = make_oracle_set(), make_b200_set()
sys.modules["qaoasim.oracle"] = _dense_oracle
sys.modules["qaoasim.kernels.numpy_impl"] = _oracle_set
sys.modules["qaoasim.kernels.numba_impl"] = _b200_set
_pkg.oracle = _dense_oracle
_kernels.numpy_impl = _oracle_set
_kernels.numba_impl = _b200_set
sys.modules["qaoasim"] = _pkg
