"""Run the reference's own test files (tests/ref/upstream/, copied byte for byte by
tests/ref/sync_reference_tests.py) against this package -- the drop-in check.

Shim, anchored on the reference's tests/conftest.py:7-11:
  * `qaoasim` and its submodules resolve to paper_2407_13012_b200 (same names);
  * the `backend` fixture runs every backend-parametrised test on BACKENDS = ("b200",);
  * `qaoasim.kernels.numpy_impl` / `numba_impl` are the oracle and a host-array
    adapter of the b200 kernel set (tests/ref/_kernel_shims.py), so
    test_kernels_parity.py checks B200 against the oracle;
  * every test is marked `gpu` (handles live in HBM);
  * SKIPS lists, with the reason, the tests that assert something only the two CPU
    kernel sets have (their names, their module objects, numba itself).
`from conftest import ...` in the copied files resolves to tests/conftest.py, whose
generators restate the reference conftest's (same streams, same instances)."""

from __future__ import annotations

import importlib
import importlib.util
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2407_13012_b200 as _pkg  # noqa: E402

BACKENDS = ("b200",)

_SUBMODULES = ("adjoint", "backend", "batch", "circuit", "cli", "costpoly", "errors", "kernels", "optimizer",
               "problems", "rng", "sampling")


def _install_alias() -> None:
    sys.modules["qaoasim"] = _pkg
    for name in _SUBMODULES:
        sys.modules[f"qaoasim.{name}"] = importlib.import_module(f"paper_2407_13012_b200.{name}")
    from _kernel_shims import make_b200_set, make_oracle_set  # noqa: E402

    oracle_set, b200_set = make_oracle_set(), make_b200_set()
    import _dense_oracle  # noqa: E402

    sys.modules["qaoasim.oracle"] = _dense_oracle
    _pkg.oracle = _dense_oracle
    sys.modules["qaoasim.kernels.numpy_impl"] = oracle_set
    sys.modules["qaoasim.kernels.numba_impl"] = b200_set
    _pkg.kernels.numpy_impl = oracle_set
    _pkg.kernels.numba_impl = b200_set


sys.path.insert(0, str(Path(__file__).resolve().parent))
_install_alias()

# `from conftest import ...` (the copied files, and this repo's own tests once this
# module holds the name) lands here: re-export every helper of tests/conftest.py, whose
# generators restate the reference conftest's (same streams, same instances)
_spec = importlib.util.spec_from_file_location("_tests_conftest", ROOT / "tests" / "conftest.py")
_base = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_base)
for _name in dir(_base):
    if not _name.startswith("_") and not _name.startswith("pytest_") and _name not in globals():
        globals()[_name] = getattr(_base, _name)

# test id (file::name, parametrisation stripped) -> why it cannot apply to a B200 drop-in
SKIPS = {
    "test_kernels_parity.py::test_samples_identical_across_paths":
        "draws through create_handle(backend_name='reference'/'accelerated'): CPU kernel-set names",
    "test_kernels_parity.py::TestSelection::test_env_flag_reference":
        "QAOA_KERNELS=reference selects the numpy CPU set, which this package replaces",
    "test_kernels_parity.py::TestSelection::test_env_flag_numpy_alias": "alias of the numpy CPU set",
    "test_kernels_parity.py::TestSelection::test_env_flag_accelerated": "selects the numba CPU set",
    "test_kernels_parity.py::TestSelection::test_auto_prefers_accelerated":
        "auto resolves to b200 here (no CPU sets); asserts the numba module",
    "test_kernels_parity.py::TestSelection::test_explicit_argument_overrides_env": "CPU set names",
}


@pytest.fixture(params=BACKENDS)
def backend(request):
    return request.param


def pytest_collection_modifyitems(config, items):
    here = Path(__file__).resolve().parent
    for item in items:
        path = Path(str(item.fspath)).resolve()
        if here not in path.parents:
            continue
        item.add_marker(pytest.mark.gpu)
        key = f"{path.name}::{'::'.join(item.nodeid.split('::')[1:]).split('[')[0]}"
        if key in SKIPS:
            item.add_marker(pytest.mark.skip(reason=f"CPU-kernel-set specific: {SKIPS[key]}"))
