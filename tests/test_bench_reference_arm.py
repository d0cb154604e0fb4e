"""bench.py's reference arm (VERDICT r01 "Next #2a"): the unmodified reference library on its own
inputs and on the reported configuration, with nothing of the product imported or mapped."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_SO = ROOT / "oracle" / "_ref" / "libdpref.so"

CHECK = r"""
import json, sys, types
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"]
sys.path.insert(0, ".")
import bench
bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"product_imported": any(m.startswith("paper_2201_01446_b200") for m in sys.modules),
                  "product_mapped": "libdpb200" in maps, "reference_mapped": "libdpref.so" in maps}))
"""


@pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built")
@pytest.mark.timeout(600)
def test_reference_arm_runs_the_reference_alone():
    r = subprocess.run([sys.executable, "-c", CHECK], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={"BENCH_REF_BUDGET_S": "1", "PATH": "/usr/bin:/bin", "OMP_NUM_THREADS": "4"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    line, probe = json.loads(lines[0]), json.loads(lines[-1])
    assert line["impl"] == "reference" and line["unit"] == "atom-steps/s" and line["value"] > 0
    assert line["config"]["same_config"] and line["config"]["atoms_total"] == 32000
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    # the reference's C2 energy on its own inputs
    assert line["reference"]["energy"] == -5040.6583216965946
    assert not probe["product_imported"] and not probe["product_mapped"] and probe["reference_mapped"]
