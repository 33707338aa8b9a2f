"""Bounds-checked build (SURVEY.md §4 T5 stand-in: compute-sanitizer is closed on this pool): every kernel
of libswof.so is rebuilt with -DSWOF_CHECK=1, whose asserts trap on any shared-memory index or global offset
outside its buffer, and tools/sanitize_case.py (cfg0, 256^2 cfg4, a variant case, fused strips, D8, the
math self-test) must run to completion under it."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_bounds_checked_build_runs_clean(gpu, tmp_path):
    from paper_1307_4839_b200 import build as b
    lib = b.build(force=True, defines=["SWOF_CHECK=1"], out=tmp_path / "libswof_checked.so")
    env = dict(os.environ, SWOF_LIB=str(lib))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_case.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "done" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    assert "check_line 0" in r.stdout, r.stdout[-2000:]
