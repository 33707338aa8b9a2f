"""The tiled stage kernel (csrc/swof_kernels.cuh: shared-memory tile) is the library's kernel in
SWOF_MARCH=0 builds.  This rebuilds the library with
SWOF_MARCH=0 and runs the one-step and predictor-stage parity tests of test_gpu_parity.py through it, in a
subprocess pointed at that build (SWOF_LIB)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_tiled_kernel_parity(gpu, tmp_path):
    from paper_1307_4839_b200 import build as b
    lib = b.build(force=True, defines=["SWOF_MARCH=0"], out=tmp_path / "libswof_tiled.so")
    env = dict(os.environ, SWOF_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-q", "-x", "-s",
                        "-k", "one_step or predictor_stage", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "10 passed" in r.stdout, r.stdout[-2000:]
    assert "'bitwise': False" not in r.stdout, r.stdout[-2000:]
