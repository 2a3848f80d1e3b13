"""Host-side logic of bench.py (no GPU): the step byte model is SURVEY.md
§8(d)'s B_fwd + B_bwd exactly, and `--gpus N` self-launches N ranks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_step_bytes_are_the_survey_formula():
    """cfg2 workload statistics of round 1 (N, N_v, F_t, P): 244.31 MB, the
    figure VERDICT r01 recomputed from SURVEY §8(d); no per-kernel double
    count (bin_fused) enters the step."""
    N, Nv, Ft, P, C = 1048576, 1016458, 1285087, 2073600, 4
    b_fwd = 16 * N + 4 * C * Nv + 16 * Ft + 4 * P * (C + 2) + 8 * P
    b_bwd = 4 * P * (C + 2) + 8 * P + 4 * Ft + (16 + 4 * C) * Nv + 4 * (C + 1) * Nv
    assert bench.step_bytes_survey(N, Nv, Ft, P, C, fwd_only=False) == b_fwd + b_bwd
    assert round((b_fwd + b_bwd) / 1e6, 2) == 244.31
    assert bench.step_bytes_survey(N, Nv, Ft, P, C, fwd_only=True) == b_fwd
    k = bench.kernel_bytes(N, Nv, Ft, P, C)
    assert k["bin_fused"] == k["project_count"] + k["scatter"]


def test_relaunch_command():
    cmd = bench.relaunch_cmd(4, ["--gpus", "4", "--steps", "3"], 29999)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == [os.path.abspath(os.path.join(ROOT, "bench.py")), "--gpus", "4", "--steps", "3"][-4:]


def test_gpus_flag_self_launches_ranks():
    """`python bench.py --gpus 2 --impl reference` (no WORLD_SIZE) re-runs
    itself under torch.distributed.run: rank 0 prints the reference line with
    n_gpus 2, rank 1 exits without work (CPU only: the reference arm is the
    oracle)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["cpu_baseline"]["kind"] == "oracle"
