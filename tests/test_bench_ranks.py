"""bench.py's multi-rank paths, launched the way the driver launches them
(python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N).

* the reference arm at N=2 (CPU only): rank 0 alone times the CPU path and
  prints ONE JSON line with impl "reference"; the other rank exits 0 silently;
* the strip and frame-stream arms at N=2 (GPU): FSR_BENCH_SINGLE_GPU=1 puts
  both ranks on cuda:0 over gloo -- a path check of the sharded bench (strip
  split, max-over-ranks timing, the final all_gather), never a measurement.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(n, args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", str(n)] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return [json.loads(l) for l in lines]


def test_reference_arm_two_ranks():
    lines = _torchrun(2, ["--impl", "reference", "--workload", "1080p", "--steps", "1",
                          "--warmup", "0", "--ref-seconds", "1"], timeout=300)
    assert len(lines) == 1, lines  # rank 0 only
    d = lines[0]
    assert d["impl"] == "reference" and d["unit"] == "fps" and d["value"] > 0
    assert d["higher_is_better"] is True and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "fps", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_strip_bench_two_ranks_on_one_gpu():
    lines = _torchrun(2, ["--workload", "1080p", "--steps", "2", "--warmup", "3", "--no-cpu"],
                      {"FSR_BENCH_SINGLE_GPU": "1"})
    assert len(lines) == 1, lines
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["unit"] == "fps"
    assert d["config"]["parallelism"] == "strips2"
    g = d["gather"]
    assert "error" not in g, g
    assert g["comm_nranks"] == 2 and g["comm_nranks_ok"] and g["own_strip_intact"]
    assert "gloo" in g["collective"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.gpu
def test_stream_bench_two_ranks_on_one_gpu():
    lines = _torchrun(2, ["--workload", "stream64", "--steps", "2", "--warmup", "3", "--no-cpu"],
                      {"FSR_BENCH_SINGLE_GPU": "1"})
    assert len(lines) == 1, lines
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "frames2"
