"""Multi-GPU domain decomposition (NCCL halo exchange) reproduces the single-GPU trajectory."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("overlap,chunk", [(True, None), (False, None), (True, "256")])
def test_two_rank_md_matches_single_gpu(tmp_path, overlap, chunk):
    out = tmp_path / "dist.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29611" if chunk else ("29614" if overlap else "29613"),
           str(ROOT / "tests" / "dist" / "dist_md_check.py"), str(out)]
    # DPB_CHECK_PLAN: every device repartition is compared with the host restatement of
    # partition_domain (domain.cpp:21-82) entry by entry; a mismatch aborts the run.
    # overlap: forward halo beside the interior chunks, reverse halo beside the owned forces
    env = dict(os.environ, DPB_CHECK_PLAN="1")
    if not overlap:
        env["DPB_NO_HALO_OVERLAP"] = "1"
    if chunk:  # several chunks per rank: interior chunks evaluated while the halo is in flight
        env["DPB_CHUNK"] = chunk
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT, env=env)
    r = json.loads(out.read_text())
    assert r["force_evals"][0] == r["force_evals"][1] == 61
    assert r["counters"][0] == r["counters"][1]
    for a, b in r["pe"]:
        assert abs(a - b) <= 1e-10 * abs(b)
    for a, b in r["ke"]:
        assert abs(a - b) <= 1e-9 * abs(b)
    assert r["pos_normwise"] <= 1e-10 and r["vel_normwise"] <= 1e-8
    assert r["pos_bitwise"] and r["vel_bitwise"], "trajectory not bitwise equal to one GPU"


@pytest.mark.skipif(n_gpus() < 4, reason="needs >= 4 GPUs")
def test_four_rank_md_matches_single_gpu(tmp_path):
    out = tmp_path / "dist4.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", "29612",
           str(ROOT / "tests" / "dist" / "dist_md_check.py"), str(out)]
    env = dict(os.environ, DPB_CHECK_PLAN="1")
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT, env=env)
    r = json.loads(out.read_text())
    assert r["world"] == 4
    for a, b in r["pe"]:
        assert abs(a - b) <= 1e-10 * abs(b)
    assert r["pos_normwise"] <= 1e-10 and r["vel_normwise"] <= 1e-8
    assert r["pos_bitwise"] and r["vel_bitwise"], "trajectory not bitwise equal to one GPU"
