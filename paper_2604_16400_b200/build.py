"""Build the collm CUDA library in-tree (sm_100a) with nvcc.

The product is a plain C-ABI shared library, ``paper_2604_16400_b200/libcollm.so`` (see
``include/collm.h``), loaded through ctypes by :mod:`paper_2604_16400_b200._lib`.  It is built
in-tree so the ``.so`` travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libcollm.so"
SOURCES = [CSRC / "collm_abi.cu"]
DEPS = sorted(CSRC.glob("*.cuh")) + [REPO_DIR / "include" / "collm.h"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-shared",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the collm CUDA library cannot be built")
    return cand


def needs_rebuild() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_rebuild():
        return LIB_PATH
    cmd = [nvcc_path(), *ARCH_FLAGS, *NVCC_FLAGS, "-I", str(REPO_DIR / "include"),
           "-o", str(LIB_PATH) + ".tmp", *map(str, SOURCES), "-lcuda"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (PKG_DIR / "build_ptxas.log").write_text(log)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{log[-6000:]}")
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    if verbose:
        print(log)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
