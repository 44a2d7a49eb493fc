"""GPU parity of the FP32 path (configs[0]: h=1, d=64, S=1024, N=4) and of the
ABI's error contract.  Calls go through the C ABI (libsppo.so) only; the
expected values come from the fp64 oracle on the same synth inputs.
Tolerance (north_star): 1e-4 for the fp32 path, allclose form (reading L7)."""

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs, ragged_offsets

pytestmark = pytest.mark.gpu

TOL = dict(atol=1e-4, rtol=1e-4)


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_10377_b200 import sppo
    c = sppo.Context(0)
    yield c
    c.close()


def run(ctx, S, h, d, offsets, window=None, dtype="fp32"):
    from paper_2503_10377_b200 import engine, sppo
    x = make_inputs(S, range(h), d, seed=S + h, dtype=torch.float32)
    dev = {k: v.cuda() for k, v in x.items()}
    L = sppo.Layout(h, d, offsets, dtype=sppo.SPPO_FP32)
    eng = engine.ChunkedAttention(ctx, L, window=window)
    out = eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ctx.sync()
    got = {k: v.cpu().double().numpy() for k, v in out.items()}
    got["lse"] = eng.lse_heads_major().cpu().double().numpy()
    xn = {k: v.double().numpy() for k, v in x.items()}
    return got, xn


def check(got, xn, offsets):
    o, lse = oracle.chunked_attention_fwd(xn["q"], xn["k"], xn["v"], offsets)
    g = oracle.chunked_attention_bwd(xn["q"], xn["k"], xn["v"], o, lse, xn["do"], offsets)
    np.testing.assert_allclose(got["o"], o, **TOL)
    np.testing.assert_allclose(got["lse"], lse, atol=1e-5, rtol=1e-5)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(got[key], g[key], **TOL, err_msg=key)


def test_config0_tiny_fp32(ctx):
    """configs[0]: 1 head, d=64, S=1024, N=4 equal chunks."""
    off = [0, 256, 512, 768, 1024]
    got, xn = run(ctx, 1024, 1, 64, off)
    check(got, xn, off)


@pytest.mark.parametrize("S,h,d,N,window", [(300, 2, 64, 5, None), (517, 3, 128, 4, 2), (129, 1, 32, 7, 3),
                                            (64, 2, 64, 1, None), (40, 1, 64, 40, 7)])
def test_fp32_ragged_windows(ctx, S, h, d, N, window):
    off = ragged_offsets(S, N, seed=S) if 1 < N < S else [round(i * S / N) for i in range(N + 1)]
    got, xn = run(ctx, S, h, d, off, window=window)
    check(got, xn, off)


def test_abi_errors(ctx):
    from paper_2503_10377_b200 import sppo
    L = sppo.Layout(1, 64, [0, 64, 128], dtype=sppo.SPPO_FP32)
    q = torch.zeros((64, 1, 64), device="cuda")
    k = torch.zeros((64, 1, 64), device="cuda")
    o = torch.zeros_like(q)
    lse = torch.zeros(64, device="cuda")

    def code(fn):
        with pytest.raises(sppo.SppoError) as e:
            fn()
        return e.value.name

    assert code(lambda: ctx.attn_fwd(L, 2, q, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_SHAPE"      # chunk out of range
    assert code(lambda: ctx.attn_fwd(L, 0, q, [1], [k], [k], o=o, lse=lse)) == "SPPO_E_SHAPE"      # id > chunk
    assert code(lambda: ctx.attn_fwd(L, 1, q, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_STATE"      # incomplete LAST
    assert code(lambda: ctx.attn_fwd(L, 1, q, [0, 0], [k, k], [k, k], o=o, lse=lse)) == "SPPO_E_STATE"  # duplicate
    assert code(lambda: ctx.attn_fwd(L, 0, None, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_ARG"
    assert code(lambda: ctx.attn_fwd(L, 1, q, [0], [k], [k], flags=sppo.SPPO_FIRST, o=o, lse=lse)) == "SPPO_E_ARG"  # no state
    bad = sppo.Layout(1, 64, [0, 64, 64], dtype=sppo.SPPO_FP32)
    assert code(lambda: ctx.attn_fwd(bad, 0, q, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_SHAPE"
    mis = torch.zeros(64 * 64 + 1, device="cuda")[1:]
    assert code(lambda: ctx.attn_fwd(L, 0, mis, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_ALIGN"
    bf = sppo.Layout(1, 64, [0, 64], dtype=sppo.SPPO_BF16)
    assert code(lambda: ctx.attn_fwd(bf, 0, q, [0], [k], [k], o=o, lse=lse)) == "SPPO_E_UNSUPPORTED"
    # non-FIRST window without an open state
    st = (torch.zeros((64, 1, 64), device="cuda"), torch.zeros(64, device="cuda"), torch.zeros(64, device="cuda"))
    assert code(lambda: ctx.attn_fwd(L, 1, q, [1], [k], [k], flags=sppo.SPPO_LAST, state=st, o=o, lse=lse)) == "SPPO_E_STATE"
    # nothing was enqueued by any failing call; a valid call still works
    ctx.attn_fwd(L, 0, q, [0], [k], [k], o=o, lse=lse)
    ctx.sync()


def test_offload_prefetch_roundtrip_bitwise(ctx):
    from paper_2503_10377_b200 import sppo
    n = 3 << 20
    src = torch.randint(-2**31, 2**31 - 1, (n // 4,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    host = ctx.host_alloc(n)
    ev = torch.cuda.Event()
    copied = ctx.kv_offload(0, src, host, n, alpha=1.0, done=ev)
    assert copied == n
    ev.synchronize()
    ctx.kv_prefetch(0, host, dst, n)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(src, dst)
    part = ctx.kv_offload(1, src, host, n, alpha=0.3)
    assert part == min(n, -(-int(np.ceil(0.3 * n)) // 65536) * 65536)
    assert ctx.kv_offload(1, src, host, n, alpha=0.0) == 0
    ctx.sync()
    ctx.host_free(host)
