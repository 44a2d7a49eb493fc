"""Degenerate and extreme cases of the bf16 path ("empty and
ragged inputs, maximum sizes, the degenerate cases the method has"):
one-token chunks (N = S), S = 1, S < one tile, a single head, chunk lengths
straddling tile boundaries, split windows of size 1; plus sampled parity at
configs[2]'s full length S = 1M on one GPU (the target workload)."""

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs, ragged_offsets

pytestmark = pytest.mark.gpu

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_10377_b200 import sppo
    c = sppo.Context(0)
    yield c
    c.close()


def run_step(ctx, S, h, off, seed, window=None):
    from paper_2503_10377_b200 import engine, sppo
    x = make_inputs(S, range(h), 128, seed=seed, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off), window=window)
    eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ctx.sync()
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    np.testing.assert_allclose(eng.lse_heads_major().double().cpu().numpy(), ref["lse"], atol=1e-3, rtol=0)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)


@pytest.mark.parametrize("S,h,off", [
    (1, 1, [0, 1]),                          # a single token
    (5, 1, [0, 1, 2, 3, 4, 5]),              # one-token chunks, N = S
    (40, 2, list(range(0, 41, 1))[::4]),     # 4-token chunks
    (127, 1, [0, 127]),                      # just under a tile
    (129, 1, [0, 128, 129]),                 # a tile plus one
    (385, 3, [0, 1, 257, 385]),              # 1-token chunk, then tile-straddling chunks
])
def test_degenerate_partitions(ctx, S, h, off):
    run_step(ctx, S, h, off, seed=S + 100)


def test_window_of_one_chunk(ctx):
    """Every prior chunk in its own window (window = 1): maximal FIRST/LAST chaining."""
    run_step(ctx, 700, 2, ragged_offsets(700, 6, seed=3), seed=77, window=1)


@pytest.mark.slow
def test_config2_full_length_sampled_parity():
    """configs[2] shape on one GPU (h=32, d=128, S=1M, N=64 equal chunks):
    sampled rows at chunk boundaries for O/LSE/dQ (2 heads) and sum_t dV_t."""
    from paper_2503_10377_b200 import engine, sppo
    from synth import make_tensor

    S, h, d, N = 1048576, 32, 128, 64
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    x = {t: make_tensor(t, S, range(h), d, seed=1, device="cuda") for t in ("q", "k", "v", "do")}
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, d, off))
    eng.step(x["q"], x["k"], x["v"], x["do"])
    torch.cuda.synchronize()
    ctx.sync()
    heads = [7, 20]
    rows = sorted({0, S - 1, 16384, 16383, 524288, 524287, 1048575 - 16384, 262144 + 77})
    host = {t: x[t][:, heads].double().cpu().numpy() for t in ("q", "k", "v", "do")}
    ref = oracle.sampled_rows(host["q"], host["k"], host["v"], rows, do=host["do"])
    lse = eng.lse_heads_major()[heads][:, rows].double().cpu().numpy()
    np.testing.assert_allclose(lse, ref["lse"], atol=1e-3, rtol=0)
    np.testing.assert_allclose(eng.o[rows][:, heads].double().cpu().numpy(), ref["o"], **O_TOL)
    np.testing.assert_allclose(eng.dq[rows][:, heads].double().cpu().numpy(), ref["dq"], **G_TOL)
    dv_sum = eng.dv[:, heads].double().sum(0).cpu().numpy()
    np.testing.assert_allclose(dv_sum, host["do"].sum(0), atol=2.0, rtol=1e-2)
    ctx.close()
