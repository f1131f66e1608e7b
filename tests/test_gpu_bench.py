"""bench.py contract on a GPU: the default line (N=1) and the multi-rank path (--gpus 2 spawns
two ranks; on a one-GPU box both share it under CKRL_BENCH_SHARE_GPU=1, which exercises the
rank spawn, the CUDA-IPC peer exchange inside the graph-captured steps and the max-over-ranks
timing — the line is marked test_mode, it is not a scaling number)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_single_gpu_line():
    j = run_bench("--steps", "7", "--warmup", "3", "--no-cpu-baseline")
    assert j["n_gpus"] == 1 and j["steps"] == 7 and j["warmup"] == 3
    assert j["roofline"]["bound"] == "hbm" and 0 < j["roofline"]["frac"] < 1.2
    assert j["e2e"]["h2d_bytes_per_step"] > 0 and j["gpu_launches"] == 14


def test_bench_two_ranks_share_gpu():
    one = run_bench("--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    two = run_bench("--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
                    env={"CKRL_BENCH_SHARE_GPU": "1"})
    assert two["n_gpus"] == 2 and "test_mode" in two
    assert two["config"]["global_envs"] == 2 * one["config"]["global_envs"]
    # rank-distinct envs: the job-wide diagnostics cover twice the units
    assert two["diagnostics"]["units"] > one["diagnostics"]["units"]


def test_bench_head_line():
    """--head: the step fed from trunk features through the tcgen05 projection (row N2)."""
    j = run_bench("--config", "cfg3", "--head", "256", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    r = j["roofline"]
    assert j["config"]["head_hidden"] == 256 and r["kernel"].startswith("proj_stats_kernel")
    assert 0 < r["tensor_frac"] < 1.2 and 0 < r["hbm_frac"] < 1.2 and r["loss_from_rows_ms_alone"] > 0
    assert j["diagnostics"]["units"] > 0


def test_bench_cfg5_variants():
    """cfg5: every {placement} x {sampler} x k variant timed, identical slabs are asserted by
    tests/test_gpu_pipeline.py; here the line's schema."""
    j = run_bench("--config", "cfg5", "--steps", "2", "--warmup", "3", "--stages", "1,2")
    keys = set(j["pipeline"])
    assert {"colocated/reference/k1", "colocated/parallel/k2", "placed/parallel/k1"} <= keys
    assert j["e2e"]["h2d_bytes_per_step"] > 0 and j["value"] > 0
