"""In-tree build of the native libraries (nvcc, sm_100a only).

  libsppo.so            — the product: C ABI (include/sppo.h) + all kernels
  tests/cuda/libtcprobe.so — test-only tcgen05/TMA layout probe
  examples/sppo_c_demo  — examples/sppo_c_demo.c: a step driven from plain C via the ABI

Run ``python -m paper_2503_10377_b200.build`` or ``__graft_entry__.build()``.
Objects are rebuilt only when a source or header is newer than the object.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]

LIB = os.path.join(PKG, "libsppo.so")
PROBE_SRC = os.path.join(ROOT, "tests", "cuda", "tc_probe.cu")
PROBE_LIB = os.path.join(ROOT, "tests", "cuda", "libtcprobe.so")
DEMO_SRC = os.path.join(ROOT, "examples", "sppo_c_demo.c")
DEMO_BIN = os.path.join(ROOT, "examples", "sppo_c_demo")  # not under build/: must ship to the GPU box


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("command failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = _headers()
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC] + FLAGS + ["-Xptxas", "-v", "-c", s, "-o", o]
            jobs.append((cmd, o + ".log"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for f in [ex.submit(_run, c, l) for c, l in jobs]:
            f.result()
    if force or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-lcudart", "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    if force or _stale(PROBE_LIB, [PROBE_SRC] + hdrs):
        _run([NVCC] + FLAGS + ["-shared", "-o", PROBE_LIB, PROBE_SRC, "-lcudart", "-Xlinker",
                               "-rpath=/usr/local/cuda/lib64"], PROBE_LIB + ".log")
    if force or _stale(DEMO_BIN, [DEMO_SRC, LIB, os.path.join(ROOT, "include", "sppo.h")]):
        _run(["gcc", "-O2", "-std=c11", "-Wall", DEMO_SRC, "-I" + os.path.join(ROOT, "include"),
              "-I/usr/local/cuda/include", "-L" + PKG, "-lsppo", "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath," + PKG + ":/usr/local/cuda/lib64", "-lm", "-o", DEMO_BIN])
    if verbose:
        for o in objs:
            log = o + ".log"
            if os.path.exists(log):
                print(open(log).read())
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
