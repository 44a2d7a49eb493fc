"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/sppo.h declares, and its host plan helpers (a0 partition, pair count,
a8 alpha) agree with the oracle.  No kernel launches (no GPU here)."""

import ctypes
import os
import re

import pytest

import oracle
from paper_2503_10377_b200 import sppo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols(name="sppo.h"):
    txt = open(os.path.join(ROOT, "include", name)).read()
    return sorted(set(re.findall(r"^\s*(?:sppo_status|const char\*|int32_t)\s+(sppo_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 14
    lib = ctypes.CDLL(sppo.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sppo.EXPORTS)
    assert sppo.lib().sppo_version() >= 100


def test_library_exports_every_layer_header_symbol():
    syms = header_symbols("sppo_layer.h")
    lib = ctypes.CDLL(sppo.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sppo.LAYER_EXPORTS)


def test_library_exports_every_pipeline_header_symbol():
    syms = header_symbols("sppo_pipeline.h")
    lib = ctypes.CDLL(sppo.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sppo.PIPELINE_EXPORTS)


def test_partition_and_pairs_match_oracle():
    for S, N in [(1024, 4), (131072, 16), (10, 3), (5, 5), (1048576, 64), (7, 1)]:
        off = sppo.partition_equal(S, N)
        assert off == oracle.offsets_from_lengths(oracle.partition_equal(S, N))
        assert sppo.causal_pairs(off) == oracle.total_pairs(off) == S * (S + 1) // 2
    with pytest.raises(sppo.SppoError) as e:
        sppo.partition_equal(3, 4)
    assert e.value.name == "SPPO_E_SHAPE"
    with pytest.raises(sppo.SppoError):
        sppo.causal_pairs([0, 5, 5])


def test_offload_alpha_matches_oracle():
    for A, m, last in [([4, 2, 1], 2, 1.0), ([2, 2, 2], 2, 1.0), ([4, 2, 1], 2, 0.0), ([0, 8, 3, 1], 4, 0.0),
                       ([1e9, 5e8, 2e8], 3e8, 1.0)]:
        assert sppo.offload_alpha(A, m, last) == pytest.approx(oracle.offload_alpha(A, m, last), abs=0, rel=1e-15)
    with pytest.raises(sppo.SppoError):
        sppo.offload_alpha([1.0], 1.0, 2.0)
    A, thr = [8.0, 6.0, 4.0, 2.0], [2.0, 3.0, 8.0, 1.0]
    assert sppo.offload_alpha(A, thr, 0.0) == oracle.offload_alpha(A, thr, 0.0) == [0.25, 0.5, 1.0, 0.0]


def test_ctx_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sppo.SppoError) as e:
        sppo.Context(0)
    assert e.value.name in ("SPPO_E_CUDA", "SPPO_E_ARG")


def test_c_demo_links_against_the_abi():
    """examples/sppo_c_demo (plain C, no torch) is built by build() and links
    libsppo.so; without a GPU it must fail loudly at sppo_ctx_create."""
    import subprocess
    import torch
    exe = os.path.join(ROOT, "examples", "sppo_c_demo")
    assert os.path.exists(exe), "run __graft_entry__.build()"
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libsppo.so" in ldd and "not found" not in ldd, ldd
    if not torch.cuda.is_available():
        r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
        assert r.returncode == 1 and "sppo_ctx_create" in r.stderr, r.stderr
