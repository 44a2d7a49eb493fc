"""Parity at the FULL sizes of every configuration bench.py times, in the
launch configuration it times (VERDICT r1 "next round" item 1):

  * C2 (configs[1]: h=32, S=128K, N=16, resident): dK/dV of EARLY keys — rows
    of chunk 0 and keys on both sides of several chunk boundaries c_j.  These
    keys receive contributions from every later chunk (P:356 [§5.1]: K_j, V_j
    take part in every later Q_i), i.e. from up to 16 backward launches summed
    into the fp32 accumulators; the oracle computes them from the definition
    (`oracle.sampled_key_grads`, one head: every row's LSE / Delta from its own
    full prefix).
  * C3 (configs[2]: h=32, S=1M, N=64, resident, 1 GPU): dK/dV of sampled keys in
    the last 4096 positions.
  * C4 (configs[3]: h=40, S=512K, N=32) under the two-level policy the bench
    times (hot prefix of 16 chunks resident, colder K/V written back and streamed
    in windows of 4, device copies poisoned with NaN after their offload).
  * C5 (configs[4]: h=64, S=4M, N=256) as one GPU's share of the 8-GPU head
    split (global heads 56..63) with FULL KV offload (hot = 0), windows of 8
    shared by 2 consecutive chunks (`--kv-group 2`), device K/V poisoned.

For the streamed configs: sampled O / LSE / dQ rows at chunk boundaries
(c_j - 1, c_j) and the last row, dK/dV of the last keys, and two identities on
the FULL tensors that hold at any size (SURVEY §8(c) "Gradient identities"):
sum_t dV_t = sum_p dO_p (rows of P sum to 1) and sum_t dK_t = 0 (adding one
vector to every key shifts each causal row uniformly).  Their tolerances are
derived in DESIGN.md ledger L19: bf16 rounding of P, dS and the stored
outputs leaves |sum| <= 2e-2 ||dK||_F per head.

Tolerances of the element checks as test_gpu_bf16 (north_star; reading L7).
Inputs: synth.make_tensor on the device (per GLOBAL head seeds), copied, never
recomputed, to the host for the oracle."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)
IDENT_REL = 2e-2  # reading L19


def _inputs(S, heads, seed):
    from synth import make_tensor
    return {t: make_tensor(t, S, heads, 128, seed=seed, device="cuda") for t in ("q", "k", "v", "do")}


def _host(x, cols, pmax=None):
    """fp32 host copies of the selected (local) head columns, rows [0, pmax)."""
    sl = slice(None) if pmax is None else slice(0, pmax)
    return {t: x[t][sl][:, cols].float().cpu().numpy() for t in ("q", "k", "v", "do")}


def _check_rows(eng, host, cols, rows):
    ref = oracle.sampled_rows(host["q"], host["k"], host["v"], rows, do=host["do"])
    lse = eng.lse_heads_major()[cols][:, rows].double().cpu().numpy()
    np.testing.assert_allclose(lse, ref["lse"], atol=1e-3, rtol=0)
    np.testing.assert_allclose(eng.o[rows][:, cols].double().cpu().numpy(), ref["o"], **O_TOL)
    np.testing.assert_allclose(eng.dq[rows][:, cols].double().cpu().numpy(), ref["dq"], **G_TOL)


def _check_keys(eng, host, cols, keys, row_block=64):
    kg = oracle.sampled_key_grads(host["q"], host["k"], host["v"], host["do"], keys, row_block=row_block)
    np.testing.assert_allclose(eng.dk[keys][:, cols].double().cpu().numpy(), kg["dk"], **G_TOL, err_msg="dk")
    np.testing.assert_allclose(eng.dv[keys][:, cols].double().cpu().numpy(), kg["dv"], **G_TOL, err_msg="dv")


def _check_identities(eng, x):
    """Per head: sum_t dV_t = sum_p dO_p and sum_t dK_t = 0 on the full tensors."""
    for h in range(eng.L.heads):
        dv, dk, do = eng.dv[:, h].double(), eng.dk[:, h].double(), x["do"][:, h].double()
        fro_v, fro_k = dv.norm().item(), dk.norm().item()
        assert (dv.sum(0) - do.sum(0)).norm().item() <= IDENT_REL * fro_v, ("sum dV", h)
        assert dk.sum(0).norm().item() <= IDENT_REL * fro_k, ("sum dK", h)
        assert torch.isfinite(dk).all() and torch.isfinite(dv).all()


def _boundary_rows(off, every):
    rows = {0, off[-1] - 1}
    for j in range(every, len(off) - 1, every):
        rows |= {off[j] - 1, off[j]}
    return sorted(rows)


def test_c2_early_key_grads_accumulated_over_all_chunks():
    """C2 resident step (the bench's headline launch configuration): dK/dV of keys
    in chunk 0 and at boundaries c_1, c_5, c_10, c_15 (accumulated over 16 - j
    backward launches) for one head, element by element against the oracle."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 131072, 32, 16
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    x = _inputs(S, range(h), seed=3)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off))
    eng.step(x["q"], x["k"], x["v"], x["do"])
    torch.cuda.synchronize()
    ctx.sync()
    cols = [13]
    keys = sorted({0, 1, 63, 127, 128, 4097, off[1] - 1} | {c for j in (1, 5, 10, 15) for c in (off[j] - 1, off[j])}
                  | {S - 1})
    _check_keys(eng, _host(x, cols), cols, keys, row_block=128)
    _check_identities(eng, x)
    ctx.close()


def test_c3_last_keys_grads():
    """C3 on one GPU (resident step as the bench times it: the forward in one
    multi-chunk launch, one persistent backward launch per chunk):
    sampled keys of the last 4096 positions (chunk 63, contributions of chunk 63
    only plus the diagonal), rows at every 16th boundary, identities."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 1048576, 32, 64
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    x = _inputs(S, range(h), seed=5)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off))
    eng.step(x["q"], x["k"], x["v"], x["do"])
    torch.cuda.synchronize()
    ctx.sync()
    cols = [29]
    host = _host(x, cols)
    keys = sorted(set(range(S - 4096, S, 331)) | {S - 4096, S - 1})
    _check_keys(eng, host, cols, keys, row_block=32)
    _check_rows(eng, host, cols, _boundary_rows(off, 16))
    _check_identities(eng, x)
    ctx.close()


def test_c4_hot_prefix_streaming_full_size():
    """C4 with the two-level policy the bench times: chunks 0..15 resident, 16..31
    written back after their forward and streamed in windows of 4; device K/V of
    cold chunks poisoned (NaN) once offloaded."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 524288, 40, 32
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    x = _inputs(S, range(h), seed=6)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, off))
    k, v = x["k"].clone(), x["v"].clone()
    stats = eng.step_kv_stream(x["q"], k, v, x["do"], hot=16, window=4, poison=True)
    torch.cuda.synchronize()
    ctx.sync()
    assert stats["h2d"] > 0
    assert torch.isnan(k[off[17]:off[18]].float()).all()  # a cold chunk really was poisoned
    del k, v
    cols = [0, 39]
    host = _host(x, cols)
    rows = _boundary_rows(off, 4)
    _check_rows(eng, host, cols, rows)
    _check_keys(eng, host, cols, sorted(set(range(S - 192, S, 13)) | {S - 1}), row_block=32)
    _check_identities(eng, x)
    eng.free_host()
    ctx.close()


def test_c5_share_full_kv_offload_grouped_full_size():
    """C5 as rank 7's share of the 8-GPU head split (global heads 56..63): full KV
    offload (hot = 0), windows of 8 chunks each serving 2 consecutive chunks,
    device K/V poisoned after their offload."""
    from paper_2503_10377_b200 import engine, sppo
    S, N = 4194304, 256
    heads = list(range(56, 64))
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    x = _inputs(S, heads, seed=8)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(len(heads), 128, off))
    k, v = x["k"].clone(), x["v"].clone()
    stats = eng.step_kv_stream_grouped(x["q"], k, v, x["do"], hot=0, window=8, group=2, poison=True)
    torch.cuda.synchronize()
    ctx.sync()
    assert stats["h2d"] > 0
    assert torch.isnan(k[off[100]:off[101]].float()).all()
    del k, v
    cols = [5]  # global head 61
    rows = _boundary_rows(off, 32)
    host = _host(x, cols)
    _check_rows(eng, host, cols, rows)
    _check_keys(eng, host, cols, sorted(set(range(S - 128, S, 17)) | {S - 1}), row_block=8)
    _check_identities(eng, x)
    eng.free_host()
    ctx.close()
