"""bench.py host-side pieces that need no GPU: the layer partitions (a0 for the
full layer: equal, attention-balanced, layer-balanced with the per-token GEMM
term), the FLOP accounting against the oracle, and the clock-rejection set."""

import argparse
import importlib.util
import os

import oracle
import oracle.layer as OL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def test_layer_partitions():
    S, N, H = 131072, 16, 4096
    eq = bench.layer_offsets(argparse.Namespace(partition="equal"), S, N, H)
    att = bench.layer_offsets(argparse.Namespace(partition="balanced"), S, N, H)
    lay = bench.layer_offsets(argparse.Namespace(partition="layer-balanced"), S, N, H)
    for off in (eq, att, lay):
        assert off[0] == 0 and off[-1] == S and len(off) == N + 1
    assert eq == oracle.offsets_from_lengths(oracle.partition_equal(S, N))
    L_att = [att[i + 1] - att[i] for i in range(N)]
    L_lay = [lay[i + 1] - lay[i] for i in range(N)]
    assert L_lay[0] < L_att[0] and L_lay[-1] > L_att[-1]  # the token-wise term evens the lengths out


def test_flop_accounting_matches_oracle():
    off = [0, 3000, 5000, 8192]
    assert bench.flops_of(off, 4, 128) == oracle.attention_flops(4, 128, off)
    f = OL.layer_flops(8192, 4096, offsets_pairs=oracle.total_pairs(off), d=128)
    assert f["gemm_fwd"] == 24 * 4096 * 4096 * 8192
    assert f["attn_fwd"] + f["attn_bwd"] == bench.flops_of(off, 32, 128)


def test_clock_reject_set():
    assert bench.CLOCK_REJECT == {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert "sw_power_cap" not in bench.CLOCK_REJECT  # kept and noted, per the timing rules


def test_bench_refuses_world_size_mismatch():
    """--gpus N must match the launcher's WORLD_SIZE (a mis-launched multi-GPU
    run would otherwise report the wrong n_gpus)."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "C1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env={**os.environ, "WORLD_SIZE": "1"})
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
