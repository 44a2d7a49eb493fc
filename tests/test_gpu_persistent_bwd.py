"""GPU parity of the persistent backward kernel's item schedule (csrc/kernels_sm100_bwd.cu,
DESIGN.md §6): the grid is one CTA pair per two SMs and the pairs take 256-key x head
items from a per-launch counter, so several items of different lengths run back to
back on each pair — K/V reloaded at each boundary, dV/dK drained by TMA reduce-add
while the next item starts.  Here a launch holds up to ~700 items (about ten per pair),
mixing full-length items with short diagonal ones and rank-1 halves of ragged pairs,
element by element against the dense fp64 oracle (tolerances of test_gpu_bf16.py,
north_star reading L7)."""

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs

pytestmark = pytest.mark.gpu

G_TOL = dict(atol=5e-2, rtol=5e-2)
O_TOL = dict(atol=2e-2, rtol=1e-2)


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_10377_b200 import sppo
    c = sppo.Context(0)
    yield c
    c.close()


def run(ctx, S, h, offsets, seed, bwd_window=None):
    from paper_2503_10377_b200 import engine, sppo
    x = make_inputs(S, range(h), 128, seed=seed, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    L = sppo.Layout(h, 128, offsets, dtype=sppo.SPPO_BF16)
    eng = engine.ChunkedAttention(ctx, L)
    eng.dk_acc.zero_()
    eng.dv_acc.zero_()
    for i in range(L.num_chunks):
        eng.forward_chunk(i, dev["q"], dev["k"], dev["v"])
    eng.window = bwd_window or 10**9
    for i in range(L.num_chunks - 1, -1, -1):
        eng.backward_chunk(i, dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ctx.sync()
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)
    return eng


@pytest.mark.parametrize("bwd_window", [None, 3])
def test_many_items_per_pair_ragged(ctx, bwd_window):
    # last chunk's launch: ceil(s_j / 256) pairs per window chunk x 28 heads ~ 700 items on
    # 74 pairs; chunk lengths not multiples of 256 (ragged pairs whose rank-1 CTA has
    # fewer than 128 or no keys), diagonal items of 1..12 Q tiles
    S, h = 3000, 28
    off = [0, 300, 1000, 1100, 2333, 3000]
    run(ctx, S, h, off, seed=21, bwd_window=bwd_window)


def test_single_tile_items(ctx):
    # 128-token chunks: every item of every launch is at most one Q tile long, so the
    # pairs turn over items (and publish the next one) on every tile
    S, h = 1024, 20
    off = [i * 128 for i in range(9)]
    run(ctx, S, h, off, seed=22)


def test_rerun_is_stable(ctx):
    # the dynamic schedule changes which pair runs which item from run to run; the fp32
    # accumulation order may differ, the result stays within a few bf16 ulps
    S, h = 2048, 24
    off = [0, 700, 1500, 2048]
    e1 = run(ctx, S, h, off, seed=23)
    dk1 = e1.dk.float().clone()
    e2 = run(ctx, S, h, off, seed=23)
    d = (e2.dk.float() - dk1).abs().max().item()
    assert d <= 2e-2 * max(1.0, dk1.abs().max().item())


@pytest.mark.parametrize("group", [1, 2, 3])
def test_grouped_multichunk_forward(ctx, group):
    # the resident step's forward as launches over groups of consecutive chunks (the
    # long-sequence schedule) equals the oracle; group 1 = per-chunk
    # multi-launch form, group 3 leaves a ragged last group
    from paper_2503_10377_b200 import engine, sppo
    S, h = 1500, 6
    off = [0, 200, 512, 700, 1024, 1300, 1500]
    x = make_inputs(S, range(h), 128, seed=30 + group, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off, dtype=sppo.SPPO_BF16), fwd_group=group)
    assert eng.fwd_multi and eng.fwd_group == group
    eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ctx.sync()
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    np.testing.assert_allclose(eng.o.double().cpu().numpy(), ref["o"], **O_TOL)
    for key in ("dq", "dk", "dv"):
        np.testing.assert_allclose(getattr(eng, key).double().cpu().numpy(), ref[key], **G_TOL, err_msg=key)
