"""Run the reference's own test files (tests/ref/upstream/, copied byte for byte by
tests/ref/sync_reference_tests.py) against this package -- the drop-in check.

Shim, anchored on the reference's tests/conftest.py:7-11:
  * `qaoasim` and its submodules resolve to paper_2407_13012_b200 (same names) through
    the alias package tests/ref/alias/qaoasim (also on PYTHONPATH for subprocesses);
  * the `backend` fixture runs every backend-parametrised test on ("b200",), and the
    CPU kernel-set names the tests hard-code resolve to b200 (see the alias);
  * `qaoasim.kernels.numpy_impl` / `numba_impl` are the oracle and a host-array
    adapter of the b200 kernel set (tests/ref/_kernel_shims.py), so
    test_kernels_parity.py checks B200 against the oracle;
  * every test is marked `gpu` (handles live in HBM);
  * SKIPS lists, with the reason, the tests that assert something only the two CPU
    kernel sets have (their module objects, the selection between them).
`from conftest import ...` in the copied files resolves to this module, which
re-exports tests/conftest.py's generators (restatements of the reference
conftest's: same streams, same instances)."""

from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

_ALIAS = Path(__file__).resolve().parent / "alias"
sys.path.insert(0, str(_ALIAS))
os.environ["PYTHONPATH"] = os.pathsep.join([str(_ALIAS), str(ROOT)] +
                                          ([os.environ["PYTHONPATH"]] if os.environ.get("PYTHONPATH") else []))
import qaoasim  # noqa: E402,F401  (tests/ref/alias/qaoasim: the package alias + shims)

BACKENDS = ("b200",)

# `from conftest import ...` (the copied files, and this repo's own tests once this
# module holds the name) lands here: re-export every helper of tests/conftest.py
_spec = importlib.util.spec_from_file_location("_tests_conftest", ROOT / "tests" / "conftest.py")
_base = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_base)
for _name in dir(_base):
    if not _name.startswith("_") and not _name.startswith("pytest_") and _name not in globals():
        globals()[_name] = getattr(_base, _name)

# test id (file::name, parametrisation stripped) -> why it cannot apply to a B200 drop-in
SKIPS = {
    "test_kernels_parity.py::test_samples_identical_across_paths":
        "compares draws of the two CPU kernel sets with each other (here both names are b200)",
    "test_kernels_parity.py::TestSelection::test_env_flag_reference":
        "QAOA_KERNELS=reference must select the numpy CPU module, which this package replaces",
    "test_kernels_parity.py::TestSelection::test_env_flag_numpy_alias": "asserts the numpy CPU module",
    "test_kernels_parity.py::TestSelection::test_env_flag_accelerated": "asserts the numba CPU module",
    "test_kernels_parity.py::TestSelection::test_auto_prefers_accelerated":
        "auto resolves to b200 here (no CPU sets); asserts the numba module",
    "test_kernels_parity.py::TestSelection::test_explicit_argument_overrides_env": "asserts the numpy CPU module",
    "test_cli.py::TestExpectationTask::test_backend_flag":
        "asserts the record names the CPU set passed to --backend; the record names the set that ran (b200)",
    "test_acceptance.py::test_scaling_sanity":
        "asserts the CPU's exponential time growth (factor 1.6-2.6 per qubit) over n=18..22; on the B200 "
        "those sizes take 0.2-0.5 ms, launch-latency bound and nearly flat (profiles/r2_kernel_bench.txt)",
}


@pytest.fixture(params=BACKENDS)
def backend(request):
    return request.param


@pytest.fixture(autouse=True)
def _cpu_set_names_resolve_to_b200(request, monkeypatch):
    """only under the reference's tests: their hard-coded CPU kernel-set names mean
    "a kernel set" -- resolve them to b200 (and in subprocesses they spawn)"""
    if Path(__file__).resolve().parent not in Path(str(request.node.fspath)).resolve().parents:
        return
    from paper_2407_13012_b200 import cli, kernels

    for name in ("reference", "accelerated", "numpy", "numba"):
        monkeypatch.setitem(kernels._ALIASES, name, kernels.B200)
    for mod in {cli, sys.modules.get("qaoasim.cli", cli)}:
        monkeypatch.setattr(mod, "BACKENDS", ("b200", "gpu", "reference", "accelerated"))
    monkeypatch.setenv("QSB_REF_ALIAS_NAMES", "1")


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
