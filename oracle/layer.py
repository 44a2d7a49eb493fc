"""fp64 oracle for one GPT transformer layer run subsequence by subsequence
 — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What is computed.  P:356 [§5.1, Fig. "computation of s_N in a Transformer-based
model and the skeletal tensors"]: the layer forward of subsequence i produces
skeletal tensors; Q_i is dead after attention, K_i/V_i are kept for later
chunks (Type-0), "the remaining 36BSH bytes of tensors" are Type-1 activations
that are offloaded with ratio alpha_i and must be back "before the backward
propagation of the subsequence begins".  The models are GPT-7B/13B/65B
(L, hidden h, heads a).  The paper does not spell the layer out;
reading L16 takes the Megatron GPT layer the paper trains on
(P:472 [§7] "implemented on top of Megatron-LM"):

    a = LN1(x)                                   LayerNorm, eps 1e-5
    q, k, v = a Wq^T + bq, a Wk^T + bk, a Wv^T + bv      (W_qkv = [Wq; Wk; Wv])
    o = CausalAttention(q, k, v)                 heads a, d = h / a (oracle/attention.py)
    y = x + o Wo^T + bo
    b = LN2(y)
    u = b W1^T + b1                              W1: [4h, h]
    g = GELU(u) = u Phi(u)                       exact (erf) GELU
    z = y + g W2^T + b2                          W2: [h, 4h]

Every op except attention acts on each token independently, so running the
layer chunk by chunk (forward i = 0..N-1, backward i = N-1..0)
is an exact rewrite of the dense layer; the chunked functions below follow that
order and accumulate the weight gradients chunk by chunk.

Backward of L = sum <dz, z> (hand-derived; pinned against torch autograd and
finite differences in tests/test_layer_oracle.py):

    dW2 = dz^T g, db2 = sum dz, dg = dz W2, du = dg * GELU'(u),
    GELU'(u) = Phi(u) + u phi(u)
    dW1 = du^T b, db1 = sum du, db = du W1, dy = dz + LN2_bwd(db)
    dWo = dy^T o, dbo = sum dy, do = dy Wo, (dq, dk, dv) = attention bwd
    dWq = dq^T a (same for k, v), da = dq Wq + dk Wk + dv Wv, dx = dy + LN1_bwd(da)
    LN_bwd: xhat = (x - mu) rstd, g = dy gamma,
            dx = rstd (g - mean(g) - xhat mean(g xhat)), dgamma = sum dy xhat, dbeta = sum dy

Layouts match the C ABI: activations token-major [S, h] (q/k/v/o viewed as
[S, a, d]), weights nn.Linear [out, in], everything float64.
"""

from __future__ import annotations

import math

import numpy as np

from .attention import causal_attention_dense_bwd, chunked_attention_bwd, chunked_attention_fwd

LN_EPS = 1e-5
_SQRT1_2 = 1.0 / math.sqrt(2.0)
_INV_SQRT_2PI = 1.0 / math.sqrt(2.0 * math.pi)

PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")

_erf = np.vectorize(math.erf, otypes=[np.float64])


def layernorm_fwd(x, gamma, beta, eps=LN_EPS):
    """Row-wise LayerNorm: returns (y, mu, rstd); mu, rstd per row."""
    x = np.asarray(x, np.float64)
    mu = x.mean(axis=1)
    var = ((x - mu[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + eps)
    y = (x - mu[:, None]) * rstd[:, None] * gamma[None, :] + beta[None, :]
    return y, mu, rstd


def layernorm_bwd(dy, x, gamma, mu, rstd):
    """Returns (dx, dgamma, dbeta) of LayerNorm (formula in the module header)."""
    xhat = (x - mu[:, None]) * rstd[:, None]
    g = dy * gamma[None, :]
    dx = rstd[:, None] * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    return dx, (dy * xhat).sum(axis=0), dy.sum(axis=0)


def gelu(u):
    """Exact GELU u * Phi(u), Phi the standard normal CDF."""
    return 0.5 * u * (1.0 + _erf(u * _SQRT1_2))


def gelu_grad(u):
    """d GELU / du = Phi(u) + u phi(u)."""
    return 0.5 * (1.0 + _erf(u * _SQRT1_2)) + u * _INV_SQRT_2PI * np.exp(-0.5 * u * u)


def _f64params(p):
    return {k: np.asarray(p[k], np.float64) for k in PARAM_NAMES}


def _chunk_fwd_pre(x, p):
    """Per-token part before attention of one chunk: LN1 and the QKV projection."""
    H = x.shape[1]
    a, mu1, rstd1 = layernorm_fwd(x, p["ln1_g"], p["ln1_b"])
    qkv = a @ p["w_qkv"].T + p["b_qkv"]
    return dict(a=a, mu1=mu1, rstd1=rstd1, q=qkv[:, :H], k=qkv[:, H:2 * H], v=qkv[:, 2 * H:])


def _chunk_fwd_post(x, o, p):
    """Per-token part after attention of one chunk: out-proj + residual, LN2, MLP."""
    y = x + o @ p["w_o"].T + p["b_o"]
    b, mu2, rstd2 = layernorm_fwd(y, p["ln2_g"], p["ln2_b"])
    u = b @ p["w_1"].T + p["b_1"]
    g = gelu(u)
    z = y + g @ p["w_2"].T + p["b_2"]
    return z, dict(y=y, b=b, mu2=mu2, rstd2=rstd2, u=u, g=g)


def layer_fwd(x, params, heads, offsets=None):
    """Layer forward.  offsets=None: dense attention; else the chunked attention
    forward over those chunk boundaries (oracle/attention.py).
    Returns (z [S,h], cache dict for layer_bwd)."""
    p = _f64params(params)
    x = np.asarray(x, np.float64)
    S, H = x.shape
    d = H // heads
    pre = _chunk_fwd_pre(x, p)
    q3, k3, v3 = (pre[t].reshape(S, heads, d) for t in ("q", "k", "v"))
    if offsets is None:
        from .attention import causal_attention_dense
        o3, lse = causal_attention_dense(q3, k3, v3)
    else:
        o3, lse = chunked_attention_fwd(q3, k3, v3, offsets)
    o = o3.reshape(S, H)
    z, post = _chunk_fwd_post(x, o, p)
    cache = dict(x=x, o=o, lse=lse, heads=heads, offsets=offsets, **pre, **post)
    return z, cache


def _zero_grads(p):
    return {k: np.zeros_like(p[k]) for k in PARAM_NAMES}


def _chunk_bwd_post(dz, c, p, gr, rows):
    """Backward of the per-token part after attention for token rows `rows`:
    returns dy (gradient at the residual stream y) and do; accumulates weight grads."""
    g, u, b, y, o = (c[t][rows] for t in ("g", "u", "b", "y", "o"))
    gr["w_2"] += dz.T @ g
    gr["b_2"] += dz.sum(axis=0)
    du = (dz @ p["w_2"]) * gelu_grad(u)
    gr["w_1"] += du.T @ b
    gr["b_1"] += du.sum(axis=0)
    dbn = du @ p["w_1"]
    dy_ln, dg2, db2 = layernorm_bwd(dbn, y, p["ln2_g"], c["mu2"][rows], c["rstd2"][rows])
    gr["ln2_g"] += dg2
    gr["ln2_b"] += db2
    dy = dz + dy_ln
    gr["w_o"] += dy.T @ o
    gr["b_o"] += dy.sum(axis=0)
    return dy, dy @ p["w_o"]


def _chunk_bwd_pre(dy, dq, dk, dv, c, p, gr, rows):
    """Backward of LN1 + QKV projection for token rows `rows`: returns dx."""
    H = dy.shape[1]
    a, x = c["a"][rows], c["x"][rows]
    dqkv = np.concatenate([dq, dk, dv], axis=1)
    gr["w_qkv"] += dqkv.T @ a
    gr["b_qkv"] += dqkv.sum(axis=0)
    da = dqkv @ p["w_qkv"]
    dx_ln, dg1, db1 = layernorm_bwd(da, x, p["ln1_g"], c["mu1"][rows], c["rstd1"][rows])
    gr["ln1_g"] += dg1
    gr["ln1_b"] += db1
    assert da.shape[1] == H
    return dy + dx_ln


def layer_bwd(dz, cache, params):
    """Dense layer backward of L = sum <dz, z>: returns (dx, grads dict)."""
    p = _f64params(params)
    dz = np.asarray(dz, np.float64)
    S, H = dz.shape
    heads = cache["heads"]
    d = H // heads
    gr = _zero_grads(p)
    allr = slice(0, S)
    dy, do = _chunk_bwd_post(dz, cache, p, gr, allr)
    q3, k3, v3 = (cache[t].reshape(S, heads, d) for t in ("q", "k", "v"))
    ab = causal_attention_dense_bwd(q3, k3, v3, do.reshape(S, heads, d))
    dq, dk, dv = (ab[t].reshape(S, H) for t in ("dq", "dk", "dv"))
    dx = _chunk_bwd_pre(dy, dq, dk, dv, cache, p, gr, allr)
    return dx, gr


def chunked_layer_bwd(dz, cache, params):
    """Layer backward in the paper's order: chunks i = N-1..0, each
    running post-attention backward, attention backward of chunk i against K/V of
    chunks 0..i (dK_j, dV_j accumulated; final after chunk j, reading L11), and
    the QKV/LN1 backward of chunk i once dK_i/dV_i are final.  Weight gradients
    accumulate over chunks.  Requires cache from layer_fwd(..., offsets)."""
    p = _f64params(params)
    dz = np.asarray(dz, np.float64)
    S, H = dz.shape
    heads, offsets = cache["heads"], list(cache["offsets"])
    d = H // heads
    N = len(offsets) - 1
    gr = _zero_grads(p)
    q3, k3, v3 = (cache[t].reshape(S, heads, d) for t in ("q", "k", "v"))
    o3 = cache["o"].reshape(S, heads, d)
    dk_acc = np.zeros((S, heads, d))
    dv_acc = np.zeros((S, heads, d))
    dx = np.zeros((S, H))
    for i in range(N - 1, -1, -1):
        r = slice(offsets[i], offsets[i + 1])
        dy, do = _chunk_bwd_post(dz[r], cache, p, gr, r)
        # attention backward of chunk i alone: dO is zero outside chunk i
        do_full = np.zeros((S, heads, d))
        do_full[r] = do.reshape(-1, heads, d)
        ab = chunked_attention_bwd(q3, k3, v3, o3, cache["lse"], do_full, offsets)
        dk_acc += ab["dk"]
        dv_acc += ab["dv"]
        dq = ab["dq"][r].reshape(-1, H)
        # dK_i, dV_i are final now: later chunks (> i) have all been processed
        dx[r] = _chunk_bwd_pre(dy, dq, dk_acc[r].reshape(-1, H), dv_acc[r].reshape(-1, H), cache, p, gr, r)
    return dx, gr


def layer_flops(S, H, offsets_pairs=None, d=128):
    """Algorithmic FLOPs of one layer fwd+bwd over S tokens:
    GEMMs 2*(3H*H + H*H + 4H*H + 4H*H) = 24 H^2 per token forward, twice that
    backward (dgrad + wgrad); attention 4d (fwd) + 10d (bwd) per causal pair per
    head, H/d heads.  offsets_pairs = total causal pairs (default S(S+1)/2)."""
    pairs = S * (S + 1) // 2 if offsets_pairs is None else offsets_pairs
    heads = H // d
    gemm = 24 * H * H * S
    return dict(gemm_fwd=gemm, gemm_bwd=2 * gemm, attn_fwd=4 * d * heads * pairs, attn_bwd=10 * d * heads * pairs)


def sampled_rows_fwd(x, params, heads, rows, block=16384):
    """Layer output z at the token rows `rows` only, for sequences too long for
    layer_fwd: LN1 and the K / V projections of every token (in row blocks),
    then for each sampled row its query, causal attention over keys 0..p (the
    definition, oracle/attention.py), out-projection, LN2 and MLP.  Pinned
    against layer_fwd on small inputs (tests/test_layer_oracle.py)."""
    p = _f64params(params)
    x = np.asarray(x, np.float64)
    S, H = x.shape
    d = H // heads
    rows = sorted(int(r) for r in rows)
    last = rows[-1] + 1
    wq, wk, wv = p["w_qkv"][:H], p["w_qkv"][H:2 * H], p["w_qkv"][2 * H:]
    bq, bk, bv = p["b_qkv"][:H], p["b_qkv"][H:2 * H], p["b_qkv"][2 * H:]
    k = np.empty((last, H))
    v = np.empty((last, H))
    for a0 in range(0, last, block):
        a1 = min(last, a0 + block)
        a, _, _ = layernorm_fwd(x[a0:a1], p["ln1_g"], p["ln1_b"])
        k[a0:a1] = a @ wk.T + bk
        v[a0:a1] = a @ wv.T + bv
    tau = 1.0 / np.sqrt(d)
    out = np.empty((len(rows), H))
    for n, r in enumerate(rows):
        a, _, _ = layernorm_fwd(x[r:r + 1], p["ln1_g"], p["ln1_b"])
        q = (a @ wq.T + bq)[0]
        o = np.empty(H)
        for h in range(heads):
            sl = slice(h * d, (h + 1) * d)
            s = tau * (k[:r + 1, sl] @ q[sl])
            w = np.exp(s - s.max())
            o[sl] = (w / w.sum()) @ v[:r + 1, sl]
        z, _ = _chunk_fwd_post(x[r:r + 1], o[None, :], p)
        out[n] = z[0]
    return rows, out
