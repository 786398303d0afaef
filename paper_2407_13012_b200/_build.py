"""Build libqsb.so (the CUDA backend) in-tree with nvcc for sm_100a.

Run as `python -m paper_2407_13012_b200._build` or through
`__graft_entry__.build()`.  Objects go to build/, the shared library next to
this file so it travels with the package.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "qsb"
LIB = PKG / "libqsb.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC,-O2,-fno-fast-math",
    "-Xptxas",
    "-v",
    f"-I{ROOT / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 backend cannot be built")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    lib_m = LIB.stat().st_mtime
    deps = _sources() + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "qsb.h"]
    return any(p.stat().st_mtime > lib_m for p in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (), lib: Path = LIB,
          objdir: Path = BUILD) -> Path:
    """defines / lib / objdir: experiment builds (tools/build_variant.py), e.g.
    defines=("QSB_EXCH_PRESYNC=1",) into a second library selected with QSB_LIB."""
    if lib == LIB and not force and not _needs_rebuild():
        return LIB
    objdir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    srcs = _sources()

    def compile_one(src: Path) -> tuple[Path, str]:
        obj = objdir / (src.stem + ".o")
        cmd = [cc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as pool:
        results = list(pool.map(compile_one, srcs))
    log = "".join(f"== {o.name}\n{e}" for o, e in results)
    (objdir / "ptxas.log").write_text(log)
    if verbose:
        sys.stderr.write(log)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results], "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
