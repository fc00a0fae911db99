"""Build libtwofold_b200.so in-tree (sm_100a): ``python -m paper_1401_6235_b200.build``."""

import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"


def build(jobs: int = 4) -> Path:
    subprocess.run(["make", "-s", "-j%d" % jobs, "-C", str(CSRC)], check=True)
    lib = CSRC.parent / "_lib" / "libtwofold_b200.so"
    if not lib.exists():
        raise RuntimeError("build did not produce %s" % lib)
    return lib


if __name__ == "__main__":
    print(build(int(sys.argv[1]) if len(sys.argv) > 1 else 4))
