"""bench.py's JSON contract on the GPU (C1, the small fp32 config): the default
head-sharded line with every required key, the context-parallel ring mode
(--parallel cp) on one rank and on two ranks sharing the one GPU (gloo)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "clocks")


def _run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_default_line_c1():
    d = _run([sys.executable, "bench.py", "--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu"])
    for k in REQUIRED + ("roofline", "e2e", "gpu_launches", "offload"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "fp32"
    assert d["roofline"]["achieved"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


def test_bench_context_parallel_one_rank_c1():
    d = _run([sys.executable, "bench.py", "--config", "C1", "--parallel", "cp", "--steps", "3", "--warmup", "3"])
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and "context parallel" in d["config"]["parallelism"]


def test_bench_context_parallel_two_ranks_one_gpu_c1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "C1",
              "--parallel", "cp", "--steps", "3", "--warmup", "3"],
             env={"SPPO_BENCH_DEVICE": "0", "SPPO_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0


def test_bench_device_budget_picks_hot_prefix_c1():
    """--device-budget: the largest KV hot prefix that fits is chosen and timed (reading L10)."""
    d = _run([sys.executable, "bench.py", "--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e",
              "--no-offload", "--device-budget", "0.0027", "--kv-window", "1"])
    b = d["kv_stream"]["budget"]
    assert 0 <= b["hot_prefix_chosen"] < 4 and b["resident_bytes"] <= 0.0027e9 < b["all_resident_bytes"]


def test_bench_plain_gpus2_self_launches_head_sharded():
    """`python bench.py --gpus 2` without torchrun launches the two ranks itself
    (here sharing the one GPU over gloo); the line reports n_gpus = 2 and the
    gathered O equals the unsharded run bit for bit (inputs are generated per
    global head and the forward is deterministic, reading L12)."""
    small = ["--config", "C2", "--heads", "4", "--seq-len", "4096", "--chunks", "4", "--steps", "3", "--warmup",
             "3", "--no-cpu", "--no-e2e", "--no-offload", "--o-digest"]
    one = _run([sys.executable, "bench.py", "--gpus", "1"] + small)
    two = _run([sys.executable, "bench.py", "--gpus", "2"] + small,
               env={"SPPO_BENCH_DEVICE": "0", "SPPO_DIST_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["heads_per_gpu"] == 2 and one["config"]["heads_per_gpu"] == 4
    assert two["gather"] is not None and two["gather"]["bytes"] == 4096 * 4 * 128 * 2
    assert one["o_sha256"] == two["o_sha256"]
