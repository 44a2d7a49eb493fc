"""Times the layer GEMMs (sppo_gemm, tcgen05) at the GPT-7B chunk shapes
against cuBLAS (torch.matmul, bf16) on the same operands.  CUDA events on the
launching stream, warm-up first; prints one JSON line per shape.

  python tools/gemm_bench.py [--tokens 8192] [--hidden 4096] [--iters 20]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10377_b200 import sppo  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    T, H = a.tokens, a.hidden
    ctx = sppo.Context(0)
    dev = "cuda"
    bf = torch.bfloat16
    shapes = [("qkv fwd", T, 3 * H, H, 0, 0), ("fc1 fwd", T, 4 * H, H, 0, 0), ("fc2 fwd", T, H, 4 * H, 0, 0),
              ("fc1 dgrad", T, H, 4 * H, 0, 1), ("fc1 wgrad", 4 * H, H, T, 1, 1), ("o wgrad", H, H, T, 1, 1)]
    for name, M, N, K, amn, bmn in shapes:
        A = torch.randn((K, M) if amn else (M, K), device=dev).to(bf)
        B = torch.randn((K, N) if bmn else (N, K), device=dev).to(bf)
        if amn:
            C = torch.zeros((M, N), device=dev)
            epi = sppo.SPPO_EPI_ACC_F32
        else:
            C = torch.empty((M, N), device=dev, dtype=bf)
            epi = sppo.SPPO_EPI_STORE
        ms = timed(lambda: ctx.gemm(M, N, K, A, B, C, a_mn=amn, b_mn=bmn, epilogue=epi), a.iters)
        At = A.t() if amn else A
        Bt = B if bmn else B.t()
        ms_cublas = timed(lambda: torch.matmul(At, Bt), a.iters)
        fl = 2.0 * M * N * K
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                          "cublas_ms": round(ms_cublas, 4), "cublas_tflops": round(fl / ms_cublas / 1e9, 1)}),
              flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
