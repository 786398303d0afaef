"""The C ABI library (libqsb.so): it loads without a GPU, exports every entry
point include/qsb.h declares, and fails loudly (no CPU fallback) when no B200
is present.  Host-only helpers are checked against Python's libm."""

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2407_13012_b200 import _lib

from conftest import HAVE_GPU, ROOT

HEADER = ROOT / "include" / "qsb.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int)\s+(qsb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_kernel_set():
    syms = header_symbols()
    for fn in ("fill_plus", "phase_by_table", "diag_scale", "rx_qubit", "weighted_probs", "probs", "tree_sum",
               "reduce_min", "reduce_max", "inner", "diag_inner", "xsum", "precompute_table", "pairwise_level"):
        assert f"qsb_{fn}" in syms


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(header_symbols()) <= set(_lib.HEADER_SYMBOLS)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_phase_lut_matches_python_libm_bitwise():
    lib = _lib.load()
    for gamma in (0.731, -1.25, 1.0 / 6.0, 3.0):
        vmin, nv = -40.0, 41
        out = np.empty(2 * nv)
        assert lib.qsb_phase_lut_host(gamma, vmin, nv, _lib.f64_ptr(out)) == 0
        for k in range(nv):
            ang = -gamma * (vmin + k)
            assert out[2 * k] == math.cos(ang) and out[2 * k + 1] == math.sin(ang)


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(RuntimeError, match="device|driver|CUDA"):
        _lib.DeviceContext(0)
    import paper_2407_13012_b200 as qs

    with pytest.raises(RuntimeError):
        qs.create_handle(qs.Polynomial(2, [(1.0, 1)]))


def test_error_mapping():
    with pytest.raises(_lib.ContractViolation):
        _lib.check(_lib.QSB_EINVAL)
    with pytest.raises(_lib.ResourceError):
        _lib.check(_lib.QSB_ENOMEM)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.QSB_ECUDA)
