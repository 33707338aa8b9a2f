"""The C ABI from plain C (examples/lake_and_dam.c): no Python and no CUDA call in the caller, host arrays in
and out.  Compiled here with gcc against include/swof.h and libswof.so; it checks well-balancedness (a lake at
rest over a bump keeps q = 0 and a flat surface to 1e-13), positivity and exact volume conservation of a
walled dam break, and exits non-zero otherwise."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_c_example_runs(gpu, tmp_path):
    from paper_1307_4839_b200 import build as b
    lib = b.build()
    exe = tmp_path / "lake_and_dam"
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-I", str(ROOT / "include"), str(ROOT / "examples" / "lake_and_dam.c"),
                    "-L", str(lib.parent), "-lswof", "-lm", f"-Wl,-rpath,{lib.parent}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
