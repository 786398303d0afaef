"""Build an experiment variant of libqsb.so with extra -D defines (A/B timing):

    python tools/build_variant.py NAME DEF=1 [DEF2=0 ...]
    QSB_LIB=paper_2407_13012_b200/libqsb_NAME.so python bench.py ...

The variant lives next to the real library (git-ignored, travels with gpurun).
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_13012_b200 import _build  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
out = _build.build(force=True, defines=defs, lib=_build.PKG / f"libqsb_{name}.so",
                   objdir=_build.ROOT / "build" / f"qsb_{name}")
print(out)
