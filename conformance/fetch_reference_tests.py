"""Stage the reference's own test suite for a conformance run (test infrastructure).

Copies /root/reference/pkg/tests/*.py into conformance/_ref_tests/ — a git-ignored directory
(like oracle/_ref: reference material stays out of history) that is NOT gpurun-ignored, so it
travels to the GPU box, where /root/reference does not exist. Run here, before `gpurun`.
"""

import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "_ref_tests"


def main() -> int:
    if not SRC.is_dir():
        print(f"{SRC} not found (the reference exists only in the build container)")
        return 1
    if DST.exists():
        shutil.rmtree(DST)
    DST.mkdir(parents=True)
    for f in sorted(SRC.glob("*.py")):
        shutil.copy2(f, DST / f.name)
    print(f"staged {len(list(DST.glob('*.py')))} files into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
