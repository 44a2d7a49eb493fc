"""Cycles per 128 x N x 128 MMA group for each operand mode (tests/cuda/tc_probe.cu),
with random-valued and all-zero operands."""
import ctypes
import os

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "cuda",
                               "libtcprobe.so"))
lib.tc_mma_bench.restype = ctypes.c_longlong
names = {0: "SS  A K-major,  B K-major ", 1: "SS  A K-major,  B MN-major", 2: "TS  A TMEM,     B MN-major",
         3: "SS  A MN-major, B MN-major", 4: "SS  A MN-major, B K-major "}
for N in (128, 64):
    for mode in range(5):
        for zero in (0, 10):
            lib.tc_mma_bench(mode + zero, N, 10)
            c = lib.tc_mma_bench(mode + zero, N, 2000)
            print(f"N={N:3d} {names[mode]} {'zeros ' if zero else 'random'}: {c} cycles per 8 MMAs (ideal {N * 4})")
