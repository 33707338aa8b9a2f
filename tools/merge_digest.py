"""Merge a digest entry written on the GPU box (gpurun_out/digest_<cfg>.json + gpurun_out/<cfg>.npz, from
tools/digest_on_box.sh) into tests/golden/."""
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
name = sys.argv[1]
ent = json.loads((ROOT / "gpurun_out" / f"digest_{name}.json").read_text())[name]
out = ROOT / "tests" / "golden" / "full_size_digests.json"
data = json.loads(out.read_text())
data[name] = ent
out.write_text(json.dumps(data, indent=1) + "\n")
shutil.copy(ROOT / "gpurun_out" / f"{name}.npz", ROOT / "tests" / "golden" / "full_size" / f"{name}.npz")
print(name, ent["steps"], ent["sha_h"][:16])
