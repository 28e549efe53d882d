"""Build libcupso.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2205_01313_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")


def build(verbose: bool = False) -> str:
    cmd = ["make", "-C", CSRC] + ([] if verbose else ["-s"])
    subprocess.run(cmd, check=True)
    return os.path.join(PKG_DIR, "libcupso.so")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
