"""The C-ABI library loads and exports every symbol include/swof.h declares; host-only entry points
(parameter validation, workspace sizing) work without a GPU.  No compute calls here."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def L():
    from paper_1307_4839_b200 import build
    build.build()
    from paper_1307_4839_b200 import lib
    return lib()


def declared_functions():
    text = (ROOT / "include" / "swof.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(swof_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("swof_create", "swof_set_state", "swof_step", "swof_run", "swof_get_state", "swof_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(L):
    from paper_1307_4839_b200 import EXPORTS
    names = declared_functions()
    assert set(names) == set(EXPORTS)
    for n in names:
        assert hasattr(L, n), n


def test_struct_layout_matches_header(L):
    """ctypes mirrors must have the C sizes (checked via a compiled probe of the header)."""
    import subprocess
    import tempfile
    from paper_1307_4839_b200.swof import SwofDiag, SwofParams
    src = '#include "swof.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu\\n", ' \
          'sizeof(swof_params), sizeof(swof_diag), offsetof(swof_params, graph_steps), offsetof(swof_diag, flags));' \
          'printf("%zu\\n", offsetof(swof_params, ga_form));}'
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "p.c"
        c.write_text(src)
        exe = Path(d) / "p"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(x) for x in out] == [C.sizeof(SwofParams), C.sizeof(SwofDiag), SwofParams.graph_steps.offset,
                                     SwofDiag.flags.offset, SwofParams.ga_form.offset]


def test_workspace_size_and_validation_on_host(L):
    from paper_1307_4839_b200 import params_from_config
    from workloads import make
    p = params_from_config(make("cfg0"))
    n = C.c_size_t()
    assert L.swof_workspace_size(C.byref(p), C.byref(n)) == 0
    # 8 fields of 64 rows x 64 doubles at minimum
    assert n.value >= 8 * 64 * 64 * 8
    bad = params_from_config(make("cfg0"))
    bad.cfl = 1.5
    assert L.swof_workspace_size(C.byref(bad), C.byref(n)) == 1
    bad = params_from_config(make("cfg0"))
    bad.bc[0] = 2      # periodic W without periodic E
    assert L.swof_workspace_size(C.byref(bad), C.byref(n)) == 1
    bad = params_from_config(make("cfg3", nx=64, ny=64))
    bad.inflow_k1[0] = 1000
    assert L.swof_workspace_size(C.byref(bad), C.byref(n)) == 1
    for field, value in (("flux", 2), ("order", 3), ("cfl_mode", 2), ("ga_form", -1)):
        bad = params_from_config(make("cfg0"))
        setattr(bad, field, value)
        assert L.swof_workspace_size(C.byref(bad), C.byref(n)) == 1, field
    assert L.swof_strerror(4) == b"out of memory"


def test_cfg4_fits_one_b200(L):
    from paper_1307_4839_b200 import params_from_config
    from workloads.configs import GreenAmpt, SwofConfig
    cfg = SwofConfig(name="cfg4", nx=8192, ny=8192, dx=1.0, dy=1.0, fric_law="manning", fric_coef=0.04, ga=GreenAmpt())
    n = C.c_size_t()
    assert L.swof_workspace_size(C.byref(params_from_config(cfg)), C.byref(n)) == 0
    assert n.value < 6e9          # ~5.4 GB of 180 GB HBM


def test_product_does_not_import_oracle():
    for f in (ROOT / "paper_1307_4839_b200").rglob("*.py"):
        assert "oracle" not in re.sub(r"#.*", "", f.read_text()).replace("never imports the oracle", ""), f
    for f in (ROOT / "paper_1307_4839_b200" / "csrc").iterdir():
        assert "swof_oracle" not in f.read_text(), f


def test_c_example_compiles_against_the_header(tmp_path):
    """examples/lake_and_dam.c (the C ABI from plain C) compiles and links against include/swof.h and
    libswof.so on a machine without a GPU (it is run by tests/test_gpu_c_example.py)."""
    import subprocess
    from paper_1307_4839_b200 import build
    lib = build.build()
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "lake_and_dam.c"), "-L", str(lib.parent), "-lswof", "-lm",
                    "-o", str(tmp_path / "lake_and_dam")], check=True)
