"""Parity at BASELINE.json's full size (configs[1], C2: h=32, d=128, S=128K,
N=16, bf16) in the launch configuration bench.py times: inputs generated on the
device (synth, torch Philox), one full fwd+bwd step through the C ABI, then
  * sampled query rows (chunk boundaries c_i, c_i - 1, first/last rows, random
    rows) for 2 heads: O_p, LSE_p, dQ_p from the oracle row by row;
  * sampled keys in the last 192 positions: dK_t, dV_t from the oracle;
  * properties on the full tensors: sum_t dV_t = sum_p dO_p per head, rows of P
    sum to 1 under the GPU's own LSE (sampled rows).
Tolerances as in test_gpu_bf16 (north_star; reading L7)."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)


def test_config1_full_size_sampled_parity():
    from paper_2503_10377_b200 import engine, sppo
    from synth import make_tensor

    S, h, d, N = 131072, 32, 128, 16
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    L = sppo.Layout(h, d, off)
    x = {t: make_tensor(t, S, range(h), d, seed=0, device="cuda") for t in ("q", "k", "v", "do")}
    eng = engine.ChunkedAttention(ctx, L)
    eng.step(x["q"], x["k"], x["v"], x["do"])
    torch.cuda.synchronize()
    ctx.sync()

    heads = [0, 31]
    g = torch.Generator().manual_seed(0)
    rows = {0, 1, 127, 128, S - 1} | {c for c in off[1:-1]} | {c - 1 for c in off[1:-1]}
    rows |= set(torch.randint(0, S, (16,), generator=g).tolist())
    rows = sorted(rows)
    pmax = rows[-1] + 1
    host = {t: x[t][:pmax, heads].double().cpu().numpy() for t in ("q", "k", "v", "do")}
    ref = oracle.sampled_rows(host["q"], host["k"], host["v"], rows, do=host["do"])
    lse = eng.lse_heads_major()[heads][:, rows].double().cpu().numpy()
    got_o = eng.o[rows][:, heads].double().cpu().numpy()
    got_dq = eng.dq[rows][:, heads].double().cpu().numpy()
    np.testing.assert_allclose(lse, ref["lse"], atol=1e-3, rtol=0)
    np.testing.assert_allclose(got_o, ref["o"], **O_TOL)
    np.testing.assert_allclose(got_dq, ref["dq"], **G_TOL)

    # rows of P sum to 1 with the GPU's LSE (O(p d) per row on the host)
    tau = 1 / np.sqrt(d)
    for n, hh in enumerate(heads):
        for r, p in enumerate(rows[:12]):
            s = tau * host["k"][: p + 1, n] @ host["q"][p, n]
            assert abs(np.exp(s - lse[n, r]).sum() - 1.0) < 2e-3

    keys = sorted(set(range(S - 192, S, 7)) | {S - 1})
    kg = oracle.sampled_key_grads(host["q"], host["k"], host["v"], host["do"], keys)
    np.testing.assert_allclose(eng.dk[keys][:, heads].double().cpu().numpy(), kg["dk"], **G_TOL)
    np.testing.assert_allclose(eng.dv[keys][:, heads].double().cpu().numpy(), kg["dv"], **G_TOL)

    # full-tensor identity: sum_t dV_t = sum_p dO_p  (rows of P sum to 1)
    dv_sum = eng.dv.double().sum(0).cpu().numpy()
    do_sum = x["do"].double().sum(0).cpu().numpy()
    np.testing.assert_allclose(dv_sum, do_sum, atol=1.0, rtol=1e-2)
    ctx.close()
