"""Pins of the full-layer oracle (oracle/layer.py) against things
other than itself: torch fp64 autograd of the layer written with torch's own
library routines (layer_norm, linear, SDPA, erf GELU), central finite
differences, GELU closed forms, LayerNorm invariants, the residual identity,
and chunked == dense for ragged chunk boundaries."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle.layer as L
import synth


def _params(H, seed=0):
    return {k: v.double().numpy() for k, v in synth.make_layer_params(H, seed, dtype=torch.float64).items()}


def _io(S, H, seed=0):
    return {k: v.double().numpy() for k, v in synth.make_layer_io(S, H, seed, dtype=torch.float64).items()}


def _torch_layer(x, p, heads):
    """The layer of the oracle header, written with torch library routines."""
    S, H = x.shape
    d = H // heads
    a = F.layer_norm(x, (H,), p["ln1_g"], p["ln1_b"], eps=1e-5)
    qkv = F.linear(a, p["w_qkv"], p["b_qkv"])
    q, k, v = (t.reshape(S, heads, d).transpose(0, 1) for t in qkv.split(H, dim=1))
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(0, 1).reshape(S, H)
    y = x + F.linear(o, p["w_o"], p["b_o"])
    b = F.layer_norm(y, (H,), p["ln2_g"], p["ln2_b"], eps=1e-5)
    return y + F.linear(F.gelu(F.linear(b, p["w_1"], p["b_1"]), approximate="none"), p["w_2"], p["b_2"])


@pytest.mark.parametrize("S,H,heads", [(24, 16, 2), (40, 32, 4)])
def test_layer_matches_torch_autograd(S, H, heads):
    p = _params(H, seed=S)
    io = _io(S, H, seed=S)
    z, cache = L.layer_fwd(io["x"], p, heads)
    dx, gr = L.layer_bwd(io["dz"], cache, p)
    tp = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    tx = torch.tensor(io["x"], requires_grad=True)
    tz = _torch_layer(tx, tp, heads)
    (tz * torch.tensor(io["dz"])).sum().backward()
    np.testing.assert_allclose(z, tz.detach().numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dx, tx.grad.numpy(), rtol=1e-10, atol=1e-12)
    for k in L.PARAM_NAMES:
        np.testing.assert_allclose(gr[k], tp[k].grad.numpy(), rtol=1e-10, atol=1e-12, err_msg=k)


def test_layer_finite_differences():
    S, H, heads = 6, 8, 2
    p = _params(H, seed=3)
    io = _io(S, H, seed=3)
    z, cache = L.layer_fwd(io["x"], p, heads)
    dx, gr = L.layer_bwd(io["dz"], cache, p)

    def loss(x=None, **over):
        pp = dict(p, **over)
        return float((L.layer_fwd(io["x"] if x is None else x, pp, heads)[0] * io["dz"]).sum())

    eps = 1e-6
    rng = np.random.default_rng(0)
    for _ in range(6):
        i, j = rng.integers(S), rng.integers(H)
        xp, xm = io["x"].copy(), io["x"].copy()
        xp[i, j] += eps
        xm[i, j] -= eps
        assert abs((loss(xp) - loss(xm)) / (2 * eps) - dx[i, j]) < 1e-7
    for name in L.PARAM_NAMES:
        w = p[name]
        idx = tuple(rng.integers(s) for s in w.shape)
        wp, wm = w.copy(), w.copy()
        wp[idx] += eps
        wm[idx] -= eps
        fd = (loss(**{name: wp}) - loss(**{name: wm})) / (2 * eps)
        assert abs(fd - gr[name][idx]) < 1e-7 * max(1.0, abs(fd)), name


def test_gelu_closed_forms():
    # GELU(u) = u Phi(u): Phi(0) = 1/2, Phi(1) = 0.8413447460685429 (standard normal table)
    u = np.array([0.0, 1.0, -1.0, 10.0, -10.0])
    np.testing.assert_allclose(L.gelu(u), [0.0, 0.8413447460685429, -0.15865525393145707, 10.0, 0.0], atol=1e-15)
    # GELU'(0) = Phi(0) = 1/2; GELU'(1) = Phi(1) + phi(1), phi(1) = exp(-1/2)/sqrt(2 pi)
    np.testing.assert_allclose(L.gelu_grad(np.array([0.0, 1.0])),
                               [0.5, 0.8413447460685429 + math.exp(-0.5) / math.sqrt(2 * math.pi)], atol=1e-15)


def test_layernorm_invariants():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(5, 64)) * 3 + 7
    y, mu, rstd = L.layernorm_fwd(x, np.ones(64), np.zeros(64))
    np.testing.assert_allclose(y.mean(axis=1), 0, atol=1e-12)
    np.testing.assert_allclose(y.var(axis=1), 1 / (1 + 1e-5 * rstd ** 2), atol=1e-12)
    y2, _, _ = L.layernorm_fwd(x + 100.0, np.ones(64), np.zeros(64))   # shift invariance
    np.testing.assert_allclose(y2, y, atol=1e-9)
    # LN backward annihilates constant row shifts and the xhat direction (dx . 1 = 0)
    dy = rng.normal(size=x.shape)
    dx, _, _ = L.layernorm_bwd(dy, x, np.ones(64), mu, rstd)
    np.testing.assert_allclose(dx.sum(axis=1), 0, atol=1e-12)


def test_residual_identity():
    """w_o = w_2 = 0, b_o = b_2 = 0: the layer is the identity and dx = dz."""
    S, H, heads = 16, 16, 2
    p = _params(H, seed=5)
    for k in ("w_o", "w_2", "b_o", "b_2"):
        p[k] = np.zeros_like(p[k])
    io = _io(S, H, seed=5)
    z, cache = L.layer_fwd(io["x"], p, heads)
    np.testing.assert_array_equal(z, io["x"])
    dx, gr = L.layer_bwd(io["dz"], cache, p)
    np.testing.assert_allclose(dx, io["dz"], atol=1e-14)
    np.testing.assert_allclose(gr["b_2"], io["dz"].sum(axis=0), atol=1e-12)
    for k in ("w_qkv", "b_qkv", "ln1_g", "ln1_b", "w_1", "b_1", "ln2_g", "ln2_b"):
        np.testing.assert_array_equal(gr[k], 0)


@pytest.mark.parametrize("offsets", [[0, 7, 19, 32], [0, 1, 2, 30, 32], [0, 32]])
def test_chunked_layer_equals_dense(offsets):
    S, H, heads = 32, 16, 2
    p = _params(H, seed=9)
    io = _io(S, H, seed=9)
    z, cache = L.layer_fwd(io["x"], p, heads)
    dx, gr = L.layer_bwd(io["dz"], cache, p)
    zc, cc = L.layer_fwd(io["x"], p, heads, offsets=offsets)
    dxc, grc = L.chunked_layer_bwd(io["dz"], cc, p)
    np.testing.assert_allclose(zc, z, atol=1e-12)
    np.testing.assert_allclose(dxc, dx, atol=1e-12)
    for k in L.PARAM_NAMES:
        np.testing.assert_allclose(grc[k], gr[k], atol=1e-11, err_msg=k)


def test_layer_flops_counts():
    f = L.layer_flops(1024, 256, d=64)
    assert f["gemm_fwd"] == 2 * (3 * 256 * 256 + 256 * 256 + 2 * 4 * 256 * 256) * 1024
    assert f["attn_fwd"] == 4 * 64 * 4 * 1024 * 1025 // 2


def test_sampled_rows_fwd_equals_dense():
    S, H, heads = 40, 16, 2
    p = _params(H, seed=13)
    io = _io(S, H, seed=13)
    z, _ = L.layer_fwd(io["x"], p, heads)
    rows, zs = L.sampled_rows_fwd(io["x"], p, heads, [0, 7, 8, 23, 39], block=16)
    np.testing.assert_allclose(zs, z[rows], rtol=1e-12, atol=1e-12)
