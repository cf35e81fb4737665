"""bench.py's multi-GPU entry (the driver's SCALE runs): --gpus must agree with
torchrun's WORLD_SIZE, --gpus N without torchrun relaunches N ranks, and the
multi-rank path prints one JSON line with n_gpus, roofline, nvlink and e2e
(on the GPU box: 2 ranks sharing its GPU over gloo)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "3"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


@pytest.mark.gpu
def test_bench_two_ranks_sharing_the_gpu(cuda_ok):
    env = dict(os.environ, SHS_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--workload", "n29", "--steps", "3",
                        "--warmup", "3", "--no-small", "--no-cpu-baseline"], env=env,
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["roofline"]["frac"] > 0 and line["nvlink"]["peak"] == 900.0
    assert line["gpu_launches"] > 0
