"""GPU tests of the two-level activation manager (reading
L8-L10): Type-1 alpha offload and KV streaming with a hot prefix, each with the
device copies poisoned (NaN) after they leave the GPU, so the backward can only
have read the bytes that came back over sppo_kv_prefetch."""

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs

pytestmark = pytest.mark.gpu

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_10377_b200 import sppo
    c = sppo.Context(0)
    yield c
    c.close()


def setup(ctx, S, h, N, seed):
    from paper_2503_10377_b200 import engine, sppo
    x = make_inputs(S, range(h), 128, seed=seed, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    L = sppo.Layout(h, 128, sppo.partition_equal(S, N))
    return x, dev, engine.ChunkedAttention(ctx, L)


def snapshot(eng):
    return {k: getattr(eng, k).clone() for k in ("o", "dq", "dk", "dv")} | {"lse": eng.lse.clone()}


def test_type1_offload_roundtrip_bitwise(ctx):
    """alpha in (0,1] prefixes of Q, O, LSE leave the GPU after fwd(i), are
    poisoned, and come back before bwd(i): O/LSE/dK/dV bitwise equal to the
    resident step (same kernels, same windows); dQ (reduce-add order) within 1 ulp-ish."""
    x, dev, eng = setup(ctx, 3072, 2, 6, seed=21)
    eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ref = snapshot(eng)
    alpha = [0.3, 0.75, 1.0, 0.5, 1.0, 0.0]
    q = dev["q"].clone()
    moved = eng.step_offload(q, dev["k"], dev["v"], dev["do"], alpha, poison=True)
    torch.cuda.synchronize()
    ctx.sync()
    assert moved["d2h"] == moved["h2d"] > 0
    for key in ("o", "lse", "dk", "dv"):
        got = getattr(eng, key)
        bad = (got != ref[key]).nonzero()
        assert bad.numel() == 0, (key, bad.shape, bad[:5].tolist(), (got.float() - ref[key].float()).abs().max().item())
    assert (eng.dq.float() - ref["dq"].float()).abs().max().item() < 1e-2
    eng.free_host()


@pytest.mark.parametrize("hot,window", [(0, 2), (2, 3), (1, 1)])
def test_kv_stream_matches_oracle(ctx, hot, window):
    S, h, N = 2048, 2, 8
    x, dev, eng = setup(ctx, S, h, N, seed=22 + hot)
    k, v = dev["k"].clone(), dev["v"].clone()
    stats = eng.step_kv_stream(dev["q"], k, v, dev["do"], hot=hot, window=window, poison=True)
    torch.cuda.synchronize()
    ctx.sync()
    assert stats["h2d"] > 0
    xn = {kk: vv.double().numpy() for kk, vv in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)
    # the device K/V of cold chunks really were poisoned
    assert torch.isnan(k[eng.L.offsets[max(hot, 0)]:eng.L.offsets[N - 2]].float()).all() or hot >= N - 2
    eng.free_host()


def test_balanced_partition_step_matches_oracle(ctx):
    """FLOPs-balanced (non-increasing, non-tile-multiple) chunks through the
    bf16 kernels, full fwd+bwd vs the dense oracle; plus the sequence-aware alpha
    offload on the same partition (bitwise round trip of O)."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 3000, 2, 5
    off = sppo.partition_balanced(S, N)
    assert off == oracle.offsets_from_lengths(oracle.partition_min_max_pairs(S, N))
    x = make_inputs(S, range(h), 128, seed=31, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off))
    eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    o_ref = eng.o.clone()
    xn = {kk: vv.double().numpy() for kk, vv in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)
    A = [eng.type1_bytes(i) for i in range(N)]
    alpha = sppo.offload_alpha(A, [A[-1]] * N, 0.0)  # constant M_threshold = the smallest chunk
    assert alpha == oracle.offload_alpha(A, [A[-1]] * N, 0.0) and alpha[0] < 1.0
    eng.step_offload(dev["q"].clone(), dev["k"], dev["v"], dev["do"], alpha, poison=True)
    torch.cuda.synchronize()
    assert torch.equal(eng.o, o_ref)
    eng.free_host()


def test_alpha_planner_in_engine_matches_oracle(ctx):
    """The bench's alpha: per-chunk M_i = BW * T_fwd(i+1) from measured forward
    times; the product's sppo_offload_alpha and the oracle agree."""
    from paper_2503_10377_b200 import sppo
    x, dev, eng = setup(ctx, 4096, 2, 4, seed=23)
    A = [eng.type1_bytes(i) for i in range(4)]
    thr = [1e6, 5e6, 2e7, 0.0]
    assert sppo.offload_alpha(A, thr, 0.0) == oracle.offload_alpha(A, thr, 0.0)


def test_host_io_step_matches_resident(ctx):
    """The e2e path bench.py times (step_host_io): Q, K, V, dO start in pinned
    host memory, the device input buffers start as NaN, and O, dQ, dK, dV end in
    pinned host memory.  Same kernels and windows as the resident step, so O,
    dK, dV are bitwise equal; dQ (reduce-add order) within 1e-2."""
    import ctypes
    x, dev, eng = setup(ctx, 2304, 2, 5, seed=24)
    eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ref = snapshot(eng)
    nb = dev["q"].numel() * dev["q"].element_size()
    host_in = {t: ctx.host_alloc(nb) for t in ("q", "k", "v", "do")}
    host_out = {t: ctx.host_alloc(nb) for t in ("o", "dq", "dk", "dv")}
    for t in host_in:
        ctx.kv_offload(0, dev[t], host_in[t], nb)
    ctx.sync()
    blank = {t: torch.full_like(dev[t], float("nan")) for t in host_in}
    h2d, d2h, last = eng.step_host_io(host_in, host_out, blank)
    last.synchronize()
    ctx.sync()
    assert h2d == 4 * nb and d2h == 4 * nb
    for t in ("o", "dq", "dk", "dv"):
        buf = (ctypes.c_uint8 * nb).from_address(host_out[t])
        got = torch.frombuffer(bytearray(buf), dtype=torch.bfloat16).view_as(ref[t])
        want = ref[t].cpu()
        if t == "dq":
            assert (got.float() - want.float()).abs().max().item() < 1e-2
        else:
            assert torch.equal(got, want), t
    for p in list(host_in.values()) + list(host_out.values()):
        ctx.host_free(p)


def test_c_demo_runs():
    """examples/sppo_c_demo: a whole step (balanced partition, fwd, O offload,
    NaN overwrite, prefetch, bwd) driven from plain C through the ABI only."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "sppo_c_demo")
    for args in ([], ["3000", "5", "3"], ["129", "2", "1"]):
        r = subprocess.run([exe] + args, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("hot,window,group", [(0, 2, 2), (2, 3, 2), (1, 2, 3), (0, 1, 4)])
def test_kv_stream_grouped_matches_oracle(ctx, hot, window, group):
    """Cold KV windows shared by `group` consecutive chunks (H2D volume / ~group),
    device K/V of cold chunks poisoned: still the dense oracle's result."""
    S, h, N = 2048, 2, 8
    x, dev, eng = setup(ctx, S, h, N, seed=40 + hot + group)
    k, v = dev["k"].clone(), dev["v"].clone()
    base = eng.step_kv_stream(dev["q"], dev["k"].clone(), dev["v"].clone(), dev["do"], hot=hot, window=window)
    stats = eng.step_kv_stream_grouped(dev["q"], k, v, dev["do"], hot=hot, window=window, group=group, poison=True)
    torch.cuda.synchronize()
    ctx.sync()
    assert 0 < stats["h2d"] < base["h2d"]
    xn = {kk: vv.double().numpy() for kk, vv in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)
    if hot < N - group - 1:
        assert torch.isnan(k[eng.L.offsets[hot]:eng.L.offsets[hot + 1]].float()).all()
    eng.free_host()
