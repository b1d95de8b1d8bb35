"""Builds the sm_100a CUDA library in-tree (csrc/Makefile -> lib/libblaz_cuda.so)."""
from __future__ import annotations

import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8) -> str:
    subprocess.check_call(["make", "-s", f"-j{jobs}", "-C", os.path.join(PKG_DIR, "csrc")])
    return os.path.join(PKG_DIR, "lib", "libblaz_cuda.so")


if __name__ == "__main__":
    print(build())
