"""Oracle timing beside the GPU numbers (SURVEY §8(d) "Oracle timing"): the fp64
numpy oracle as it stands, on this host's cores (all BLAS threads, and 1
thread), for C1 in full and for a medium point (1 head, d=128, S=16384, N=4);
the measured pair rate extrapolated to the full configs (labelled as
extrapolation).  Test/measurement tool: it runs only oracle/ code.
usage: python tools/oracle_timing.py > profiles/r01/oracle_timing.json"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from threadpoolctl import threadpool_limits, threadpool_info  # noqa: E402

import oracle  # noqa: E402
from synth import make_inputs  # noqa: E402

CONFIGS = {"C1": (1, 64, 1024, 4), "C2": (32, 128, 131072, 16), "C3": (32, 128, 1048576, 64),
           "C4": (40, 128, 524288, 32), "C5": (64, 128, 4194304, 256)}


def flops(h, d, S):
    return 14 * d * h * S * (S + 1) // 2


def run(h, d, S, N, dtype):
    x = make_inputs(S, range(h), d, seed=0, dtype=dtype)
    off = oracle.offsets_from_lengths(oracle.partition_equal(S, N))
    t = 0.0
    for hh in range(h):
        xn = {k: v[:, hh:hh + 1].double().numpy() for k, v in x.items()}
        t0 = time.perf_counter()
        o, lse = oracle.chunked_attention_fwd(xn["q"], xn["k"], xn["v"], off)
        oracle.chunked_attention_bwd(xn["q"], xn["k"], xn["v"], o, lse, xn["do"], off)
        t += time.perf_counter() - t0
    return t


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


out = {"cpu_model": cpu_model(), "cores_affinity": len(os.sched_getaffinity(0)),
       "blas": [{k: t.get(k) for k in ("internal_api", "num_threads")} for t in threadpool_info()]}
meas = {}
for label, threads in (("all_threads", None), ("1_thread", 1)):
    with threadpool_limits(limits=threads):
        c1 = run(*CONFIGS["C1"], torch.float32)
        med = run(1, 128, 16384, 4, torch.bfloat16)
    fl_med = flops(1, 128, 16384)
    meas[label] = {"C1_full_s": round(c1, 3), "C1_tflops": flops(1, 64, 1024) / c1 / 1e12,
                   "medium_s": round(med, 2), "medium_tflops": fl_med / med / 1e12,
                   "medium": "1 head, d=128, S=16384, N=4, fwd+bwd"}
out["measured"] = meas
rate = {k: v["medium_tflops"] * 1e12 for k, v in meas.items()}
out["extrapolated_full_oracle_hours"] = {
    c: {k: round(flops(h, d, S) / r / 3600, 2) for k, r in rate.items()}
    for c, (h, d, S, N) in CONFIGS.items() if c != "C1"}
out["note"] = "extrapolation = config FLOPs / medium-point rate (the oracle's cost is the same 14 d FLOP per causal pair)"
print(json.dumps(out, indent=1))
