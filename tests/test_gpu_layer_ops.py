"""GPU parity of the per-chunk layer's building blocks through the C ABI
(include/sppo_layer.h): the tcgen05 GEMM in its three orientations (forward
x W^T, data gradient dy W, weight gradient dy^T x accumulated in fp32), its
fused epilogues (bias, residual, GELU with saved pre-activation, GELU
backward, split operands / outputs), LayerNorm forward / backward and the
column reductions — each against fp64 references on the same bf16 values
(matmul as the library primitive; GELU / LayerNorm from oracle/layer.py).

Tolerances: bf16 outputs carry one RNE rounding (relative 2^-9) on top of an
fp32-accumulated sum, so |gpu - ref| <= 1e-2 |ref| + 1e-2 * rms(ref) holds with
margin; fp32 weight-gradient accumulators carry only the fp32 summation error."""

import numpy as np
import pytest
import torch

import oracle.layer as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_10377_b200 import sppo
    c = sppo.Context(0)
    yield c
    c.close()


def _rand(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * std).to(torch.bfloat16)


def _np(t):
    return t.double().cpu().numpy()


def _close(got, ref, rtol=1e-2, ftol=1e-2, what=""):
    got = _np(got) if isinstance(got, torch.Tensor) else got
    scale = np.sqrt(np.mean(ref ** 2)) + 1e-30
    err = np.abs(got - ref)
    bound = rtol * np.abs(ref) + ftol * scale
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} outside tolerance, max err {err.max():.3e} (rms {scale:.3e})"


@pytest.mark.parametrize("M,N,K", [(300, 512, 320), (128, 384, 64), (1000, 256, 1000), (17, 128, 8)])
def test_gemm_forward_bias_residual(ctx, M, N, K):
    from paper_2503_10377_b200 import sppo
    x, w, b, r = _rand((M, K), 1), _rand((N, K), 2, 0.05), _rand((N,), 3), _rand((M, N), 4)
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    xd, wd, bd, rd = x.cuda(), w.cuda(), b.cuda(), r.cuda()
    ctx.gemm(M, N, K, xd, wd, c, bias=bd, residual=rd)
    ref = _np(x) @ _np(w).T + _np(b) + _np(r)
    _close(c, ref, what="x W^T + b + r")
    ctx.gemm(M, N, K, xd, wd, c, epilogue=sppo.SPPO_EPI_STORE)
    _close(c, _np(x) @ _np(w).T, what="x W^T")


@pytest.mark.parametrize("M,N,K", [(256, 384, 512), (200, 256, 136)])
def test_gemm_data_gradient(ctx, M, N, K):
    dy, w = _rand((M, K), 5), _rand((K, N), 6, 0.05)  # B stored [K][N] (the weight [out][in], out = K)
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.gemm(M, N, K, dy.cuda(), w.cuda(), c, b_mn=1)
    _close(c, _np(dy) @ _np(w), what="dy W")


@pytest.mark.parametrize("M,N,K", [(384, 256, 200), (128, 512, 1024)])
def test_gemm_weight_gradient_accumulates(ctx, M, N, K):
    from paper_2503_10377_b200 import sppo
    dy, x = _rand((K, M), 7), _rand((K, N), 8)  # A stored [K][M] (dy [tokens][out]), B stored [K][N]
    acc0 = torch.randn((M, N), generator=torch.Generator().manual_seed(9))
    acc = acc0.clone().cuda()
    for _ in range(2):
        ctx.gemm(M, N, K, dy.cuda(), x.cuda(), acc, a_mn=1, b_mn=1, epilogue=sppo.SPPO_EPI_ACC_F32)
    ref = acc0.double().numpy() + 2 * (_np(dy).T @ _np(x))
    _close(acc, ref, rtol=1e-4, ftol=1e-5, what="acc += dy^T x")


def test_gemm_split_operands_and_outputs(ctx):
    """QKV: C split into three [M, H] outputs; dQKV: K-major A from three parts;
    wgrad of QKV: M-major A from three parts."""
    from paper_2503_10377_b200 import sppo
    M, H = 256, 256
    a, w = _rand((M, H), 10), _rand((3 * H, H), 11, 0.05)
    outs = [torch.empty((M, H), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    ctx.gemm(M, 3 * H, H, a.cuda(), w.cuda(), outs)
    ref = _np(a) @ _np(w).T
    for i in range(3):
        _close(outs[i], ref[:, i * H:(i + 1) * H], what=f"qkv part {i}")
    parts = [_rand((M, H), 20 + i) for i in range(3)]
    da = torch.empty((M, H), dtype=torch.bfloat16, device="cuda")
    ctx.gemm(M, H, 3 * H, [p.cuda() for p in parts], w.cuda(), da, b_mn=1)
    cat = np.concatenate([_np(p) for p in parts], axis=1)
    _close(da, cat @ _np(w), what="[dq dk dv] W_qkv")
    dw = torch.zeros((3 * H, H), device="cuda")
    ctx.gemm(3 * H, H, M, [p.cuda() for p in parts], a.cuda(), dw, a_mn=1, b_mn=1, epilogue=sppo.SPPO_EPI_ACC_F32)
    _close(dw, cat.T @ _np(a), rtol=1e-4, ftol=1e-5, what="[dq dk dv]^T a")


def test_gemm_gelu_and_dgelu_epilogues(ctx):
    from paper_2503_10377_b200 import sppo
    M, N, K = 384, 1024, 256
    x, w, b = _rand((M, K), 12), _rand((N, K), 13, 0.1), _rand((N,), 14)
    g = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    u = torch.empty_like(g)
    ctx.gemm(M, N, K, x.cuda(), w.cuda(), g, bias=b.cuda(), aux_out=u, epilogue=sppo.SPPO_EPI_GELU)
    uref = _np(x) @ _np(w).T + _np(b)
    _close(u, uref, what="pre-activation u")
    _close(g, L.gelu(uref), what="GELU(u)")
    # backward through the GELU: du = (dz W2) * GELU'(u) with the stored bf16 u
    K2 = 512
    dz, w2 = _rand((M, K2), 15), _rand((K2, N), 16, 0.05)
    du = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.gemm(M, N, K2, dz.cuda(), w2.cuda(), du, b_mn=1, aux_in=u, epilogue=sppo.SPPO_EPI_DGELU)
    _close(du, (_np(dz) @ _np(w2)) * L.gelu_grad(_np(u)), what="dGELU")


def test_gemm_rejects_bad_shapes(ctx):
    from paper_2503_10377_b200 import sppo
    a = torch.zeros((128, 64), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((100, 64), dtype=torch.bfloat16, device="cuda")
    c = torch.zeros((128, 100), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(sppo.SppoError) as e:
        ctx.gemm(128, 100, 64, a, w, c)
    assert e.value.name == "SPPO_E_SHAPE"
    with pytest.raises(sppo.SppoError) as e:
        ctx.gemm(128, 128, 64, a, w, c, epilogue=sppo.SPPO_EPI_GELU)
    assert e.value.name == "SPPO_E_ARG"


@pytest.mark.parametrize("rows,cols", [(300, 512), (64, 4096)])
def test_layernorm_forward_backward_and_param_grads(ctx, rows, cols):
    x = _rand((rows, cols), 30, 2.0) + 3
    gam, bet = 1 + 0.1 * _rand((cols,), 31).float(), 0.1 * _rand((cols,), 32).float()
    gam, bet = gam.to(torch.bfloat16), bet.to(torch.bfloat16)
    y = torch.empty((rows, cols), dtype=torch.bfloat16, device="cuda")
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    xd = x.cuda()
    ctx.layernorm_fwd(xd, gam.cuda(), bet.cuda(), y, mean, rstd)
    yref, mref, rref = L.layernorm_fwd(_np(x), _np(gam), _np(bet))
    _close(y, yref, what="LN y")
    np.testing.assert_allclose(mean.double().cpu().numpy(), mref, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(rstd.double().cpu().numpy(), rref, rtol=1e-4)
    dy, dres = _rand((rows, cols), 33), _rand((rows, cols), 34)
    dx = torch.empty_like(y)
    ctx.layernorm_bwd(dy.cuda(), xd, gam.cuda(), mean, rstd, dx, dres=dres.cuda())
    dxref, dgref, dbref = L.layernorm_bwd(_np(dy), _np(x), _np(gam), mref, rref)
    _close(dx, dxref + _np(dres), what="LN dx + dres")
    dg = torch.zeros(cols, device="cuda")
    db = torch.zeros(cols, device="cuda")
    ctx.col_reduce(dy.cuda(), rows, cols, db, x=xd, mean=mean, rstd=rstd, prod_acc=dg)
    _close(dg, dgref, rtol=1e-3, ftol=1e-4, what="dgamma")
    _close(db, dbref, rtol=1e-3, ftol=1e-4, what="dbeta")


def test_col_reduce_split_parts(ctx):
    rows, H = 1000, 256
    parts = [_rand((rows, H), 40 + i) for i in range(3)]
    acc = torch.ones(3 * H, device="cuda")
    ctx.col_reduce([p.cuda() for p in parts], rows, 3 * H, acc)
    ref = 1 + np.concatenate([_np(p).sum(axis=0) for p in parts])
    _close(acc, ref, rtol=1e-4, ftol=1e-5, what="bias grad over 3 parts")


def test_col_reduce_narrow_parts_and_ragged_width(ctx):
    """Parts of 128 columns (a tensor-parallel QKV gradient) and widths that are not
    a multiple of 256."""
    rows = 300
    parts = [_rand((rows, 128), 50 + i) for i in range(3)]
    acc = torch.zeros(384, device="cuda")
    ctx.col_reduce([p.cuda() for p in parts], rows, 384, acc)
    _close(acc, np.concatenate([_np(p).sum(axis=0) for p in parts]), rtol=1e-4, ftol=1e-5, what="3 x 128")
    x = _rand((rows, 136), 60)
    acc = torch.zeros(136, device="cuda")
    ctx.col_reduce(x.cuda(), rows, 136, acc)
    _close(acc, _np(x).sum(axis=0), rtol=1e-4, ftol=1e-5, what="width 136")
