"""Copy the reference's own test files (/root/reference/pkg/tests/test_*.py) into
tests/ref/upstream/ so pytest runs them against this package (tests/ref/conftest.py
maps `qaoasim` onto paper_2407_13012_b200 with BACKENDS = ("b200",)).

The copies are git-ignored -- the reference's tests are not part of this repo's
history -- but travel to the GPU box with the working tree (gpurun snapshots it).
Files are copied byte for byte; nothing in them is edited.  Their
`from conftest import ...` helpers resolve to tests/conftest.py, which restates the
reference conftest's generators (same streams, same instances).

    python tests/ref/sync_reference_tests.py [REFERENCE_TESTS_DIR]
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
DEST = HERE / "upstream"


def sync(src: Path) -> list[str]:
    DEST.mkdir(exist_ok=True)
    copied = []
    for f in sorted(src.glob("test_*.py")):
        shutil.copyfile(f, DEST / f.name)
        copied.append(f.name)
    return copied


if __name__ == "__main__":
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else Path("/root/reference/pkg/tests")
    names = sync(src)
    print(f"copied {len(names)} reference test files into {DEST}: {', '.join(names)}")
