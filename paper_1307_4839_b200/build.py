"""Build libswof.so (the C-ABI library, include/swof.h) in-tree for sm_100a with nvcc.

libswof.so is the bit-identical build (-DSWOF_EXACT=1 -fmad=false): no multiply-add contraction, the
evaluation order of every expression is the canonical sheet of DESIGN.md §3, division and sqrt IEEE
(nvcc defaults: -prec-div=true -prec-sqrt=true -ftz=false).  tolerance=True builds the measured-and-rejected
tolerance-contract variant (-DSWOF_EXACT=0 -fmad=true; DESIGN.md §3 "contract") into another file, for
A/B experiments only.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libswof.so"
SOURCES = [CSRC / "swof.cu"]
DEPS = SOURCES + [CSRC / "swof_kernels.cuh", CSRC / "swof_d8.cuh", CSRC / "swof_march.cuh", ROOT / "include" / "swof.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
    "-I", str(ROOT / "include"),
]


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, defines=(), out: Path = None, tolerance: bool = False) -> Path:
    """Compile the library (out: another file for a diagnostic build, e.g. -DSWOF_CHECK=1, or for the
    tolerance=True experiment)."""
    out = Path(out) if out is not None else LIB
    if tolerance and out == LIB:
        raise ValueError("the tolerance-contract variant is an experiment: build it into another file")
    if out == LIB and not force and not stale(out):
        return out
    tmp = out.with_suffix(f".so.tmp{os.getpid()}")
    extra = os.environ.get("SWOF_NVCC_EXTRA", "").split()        # A/B experiments (tools/ab.sh) only
    mode = ["-DSWOF_EXACT=0", "-fmad=true"] if tolerance else ["-DSWOF_EXACT=1", "-fmad=false"]
    cmd = [NVCC, *NVCC_FLAGS, *mode, *extra, *[f"-D{d}" for d in defines], "-o", str(tmp), *map(str, SOURCES),
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}): {' '.join(cmd)}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    if out == LIB:
        (PKG / "libswof.ptxas.txt").write_text(r.stderr)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True,
                defines=[a[2:] for a in sys.argv[1:] if a.startswith("-D")]))
