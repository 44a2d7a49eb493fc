"""Pins for the fp64 oracle (CPU only).  Each test checks the oracle against
something other than itself: a library routine (torch SDPA + autograd in fp64),
closed forms, invariants, finite differences, brute force on tiny inputs, and the
SPEC's worked examples in tests/golden/.  A plausible slip in the oracle (dropped
term, wrong sign/index, transposed operand, off-by-one mask) fails at least one.
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs, ragged_offsets

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def rnd(S, h, d, seed=0):
    t = make_inputs(S, range(h), d, seed=seed, dtype=torch.float32)
    return {k: v.double().numpy() for k, v in t.items()}


def sdpa_ref(q, k, v, do, scale):
    """torch's own causal SDPA + autograd in fp64 (library routine pin)."""
    tq, tk, tv = (torch.tensor(x.transpose(1, 0, 2), requires_grad=True) for x in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True, scale=scale)
    o.backward(torch.tensor(do.transpose(1, 0, 2)))
    tr = lambda x: x.detach().numpy().transpose(1, 0, 2)
    return tr(o), tr(tq.grad), tr(tk.grad), tr(tv.grad)


# --------------------------------------------------------------- dense pins

@pytest.mark.parametrize("S,h,d", [(1, 1, 4), (7, 2, 8), (64, 3, 16), (200, 1, 64)])
def test_dense_matches_torch_sdpa_and_autograd(S, h, d):
    x = rnd(S, h, d, seed=S)
    ref = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], x["do"])
    o, dq, dk, dv = sdpa_ref(x["q"], x["k"], x["v"], x["do"], 1 / np.sqrt(d))
    np.testing.assert_allclose(ref["o"], o, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ref["dq"], dq, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(ref["dk"], dk, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(ref["dv"], dv, rtol=1e-10, atol=1e-12)


def test_dense_lse_is_logsumexp_of_causal_row():
    from scipy.special import logsumexp
    x = rnd(50, 2, 8, seed=3)
    _, lse = oracle.causal_attention_dense(x["q"], x["k"], x["v"])
    tau = 1 / np.sqrt(8)
    for hh in range(2):
        for p in range(50):
            s = tau * x["k"][: p + 1, hh] @ x["q"][p, hh]
            assert abs(lse[hh, p] - logsumexp(s)) < 1e-12


def test_closed_form_q_zero():
    """Q = 0 => uniform weights over t <= p: O_p = mean(v_0..v_p), LSE_p = ln(p+1)."""
    x = rnd(40, 2, 8, seed=4)
    q = np.zeros_like(x["q"])
    o, lse = oracle.causal_attention_dense(q, x["k"], x["v"])
    cum = np.cumsum(x["v"], axis=0) / np.arange(1, 41)[:, None, None]
    np.testing.assert_allclose(o, cum, atol=1e-13)
    np.testing.assert_allclose(lse, np.log(np.arange(1, 41))[None, :].repeat(2, 0), atol=1e-13)


def test_closed_form_row0_and_constant_v_and_convex_hull():
    x = rnd(33, 2, 8, seed=5)
    o, lse = oracle.causal_attention_dense(x["q"], x["k"], x["v"])
    np.testing.assert_allclose(o[0], x["v"][0], atol=1e-14)                      # row 0 sees only key 0
    np.testing.assert_allclose(lse[:, 0], np.einsum("hd,hd->h", x["q"][0], x["k"][0]) / np.sqrt(8), atol=1e-14)
    vmin = np.minimum.accumulate(x["v"], axis=0)
    vmax = np.maximum.accumulate(x["v"], axis=0)
    assert np.all(o >= vmin - 1e-12) and np.all(o <= vmax + 1e-12)              # convex combination
    c = np.full_like(x["v"], 0.37)
    g = oracle.causal_attention_dense_bwd(x["q"], x["k"], c, x["do"])
    np.testing.assert_allclose(g["o"], c, atol=1e-14)
    assert np.abs(g["dq"]).max() < 1e-13 and np.abs(g["dk"]).max() < 1e-13


def test_rows_of_p_sum_to_one():
    x = rnd(64, 2, 16, seed=6)
    _, lse = oracle.causal_attention_dense(x["q"], x["k"], x["v"])
    tau = 1 / 4.0
    for hh in range(2):
        s = tau * x["q"][:, hh] @ x["k"][:, hh].T
        p = np.where(np.tril(np.ones((64, 64), bool)), np.exp(s - lse[hh][:, None]), 0)
        np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-13)


def test_finite_difference_gradients():
    """Central FD on L = sum <dO, O>, h=1, S=12, d=4."""
    x = rnd(12, 1, 4, seed=7)
    g = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], x["do"])

    def L(which):
        def f(arr):
            args = dict(q=x["q"], k=x["k"], v=x["v"])
            args[which] = arr
            o, _ = oracle.causal_attention_dense(args["q"], args["k"], args["v"])
            return float((o * x["do"]).sum())
        return f

    for name, key in (("q", "dq"), ("k", "dk"), ("v", "dv")):
        fd = oracle.fd_grad(L(name), x[name])
        np.testing.assert_allclose(g[key], fd, rtol=1e-6, atol=1e-8)


def test_gradient_identities():
    """sum_t dK_t = 0 (shift of all keys is a per-row constant); sum_t dV_t = sum_p dO_p
    (rows of P sum to 1); sum_t P_pt dP_pt = Delta_p."""
    x = rnd(96, 3, 16, seed=8)
    g = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], x["do"])
    np.testing.assert_allclose(g["dk"].sum(0), 0.0, atol=1e-12)
    np.testing.assert_allclose(g["dv"].sum(0), x["do"].sum(0), atol=1e-12)
    zero = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], np.zeros_like(x["do"]))
    for key in ("dq", "dk", "dv"):
        assert np.abs(zero[key]).max() == 0.0
    tau = 0.25
    for hh in range(3):
        s = tau * x["q"][:, hh] @ x["k"][:, hh].T
        p = np.where(np.tril(np.ones((96, 96), bool)), np.exp(s - g["lse"][hh][:, None]), 0)
        dp = x["do"][:, hh] @ x["v"][:, hh].T
        np.testing.assert_allclose((p * dp).sum(1), g["delta"][hh], atol=1e-12)


# --------------------------------------------------------------- chunked pins

@pytest.mark.parametrize("S,h,d,N", [(16, 1, 4, 1), (37, 2, 8, 3), (64, 1, 64, 4), (100, 2, 8, 7), (24, 1, 4, 24)])
def test_chunked_equals_dense(S, h, d, N):
    x = rnd(S, h, d, seed=S + N)
    off = ragged_offsets(S, N, seed=N) if N not in (1, S) else list(range(0, S + 1, S // N))
    o_ref, lse_ref = oracle.causal_attention_dense(x["q"], x["k"], x["v"])
    o, lse = oracle.chunked_attention_fwd(x["q"], x["k"], x["v"], off)
    np.testing.assert_allclose(o, o_ref, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, atol=1e-12)
    g_ref = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], x["do"])
    g = oracle.chunked_attention_bwd(x["q"], x["k"], x["v"], o, lse, x["do"], off)
    for key in ("dq", "dk", "dv", "delta"):
        np.testing.assert_allclose(g[key], g_ref[key], atol=1e-11)


def test_n_invariance():
    x = rnd(120, 2, 8, seed=9)
    outs = []
    for N in (1, 2, 5, 8, 120):
        off = [round(i * 120 / N) for i in range(N + 1)]
        o, lse = oracle.chunked_attention_fwd(x["q"], x["k"], x["v"], off)
        g = oracle.chunked_attention_bwd(x["q"], x["k"], x["v"], o, lse, x["do"], off)
        outs.append((o, lse, g["dq"], g["dk"], g["dv"]))
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            np.testing.assert_allclose(a, b, atol=1e-12)


def test_window_split_and_merge_algebra():
    x = rnd(60, 2, 8, seed=10)
    off = [0, 11, 29, 30, 60]
    o_ref, lse_ref = oracle.chunked_attention_fwd(x["q"], x["k"], x["v"], off)
    windows = [[[0]], [[1], [0]], [[2, 0], [1]], [[3], [1, 2], [0]]]
    o, lse = oracle.chunked_attention_fwd_windows(x["q"], x["k"], x["v"], off, windows)
    np.testing.assert_allclose(o, o_ref, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, atol=1e-12)
    with pytest.raises(ValueError):
        oracle.chunked_attention_fwd_windows(x["q"], x["k"], x["v"], off, [[[0]], [[1]], [[0, 1, 2]], [[3]]])
    # merge: identity, commutativity, associativity
    rng = np.random.default_rng(0)
    mk = lambda: (rng.normal(size=(5, 2, 3)), rng.normal(size=(2, 5)), rng.uniform(0.5, 2, size=(2, 5)))
    a, b, c = mk(), mk(), mk()
    e = oracle.empty_state(5, 2, 3)
    for u, w in zip(oracle.merge_states(a, e), a):
        np.testing.assert_allclose(u, w, atol=1e-15)
    for u, w in zip(oracle.merge_states(a, b), oracle.merge_states(b, a)):
        np.testing.assert_allclose(u, w, atol=1e-14)
    for u, w in zip(oracle.merge_states(oracle.merge_states(a, b), c), oracle.merge_states(a, oracle.merge_states(b, c))):
        np.testing.assert_allclose(u, w, atol=1e-13)
    # finalize of merged == softmax over the union (brute force on 2 scalar blocks)
    s1, s2 = np.array([0.3, -1.2]), np.array([2.0])
    v1, v2 = np.array([[1.0], [2.0]]), np.array([[5.0]])
    st = lambda s, v: ((np.exp(s - s.max()) @ v)[None, None, :], np.array([[s.max()]]), np.array([[np.exp(s - s.max()).sum()]]))
    o, lse = oracle.finalize_state(oracle.merge_states(st(s1, v1), st(s2, v2)))
    sa = np.concatenate([s1, s2])
    w = np.exp(sa) / np.exp(sa).sum()
    assert abs(o[0, 0, 0] - w @ np.array([1.0, 2.0, 5.0])) < 1e-14
    assert abs(lse[0, 0] - np.log(np.exp(sa).sum())) < 1e-14


def test_sampled_rows_and_key_grads_match_dense():
    x = rnd(300, 2, 16, seed=11)
    g = oracle.causal_attention_dense_bwd(x["q"], x["k"], x["v"], x["do"])
    rows = [0, 1, 127, 128, 255, 299]
    r = oracle.sampled_rows(x["q"], x["k"], x["v"], rows, do=x["do"])
    np.testing.assert_allclose(r["o"], g["o"][rows], atol=1e-12)
    np.testing.assert_allclose(r["lse"], g["lse"][:, rows], atol=1e-12)
    np.testing.assert_allclose(r["delta"], g["delta"][:, rows], atol=1e-12)
    np.testing.assert_allclose(r["dq"], g["dq"][rows], atol=1e-12)
    # late keys, and early keys (rows of blocks that precede some keys: P = 0 there)
    for keys, rb in (([250, 251, 299], 17), ([0, 1, 16, 17, 100, 299], 7), ([3, 150], 300), ([299], 1)):
        kg = oracle.sampled_key_grads(x["q"], x["k"], x["v"], x["do"], keys, row_block=rb)
        np.testing.assert_allclose(kg["dk"], g["dk"][keys], atol=1e-12)
        np.testing.assert_allclose(kg["dv"], g["dv"][keys], atol=1e-12)
    r1 = oracle.sampled_rows(x["q"], x["k"], x["v"], [5], heads=[1])
    np.testing.assert_allclose(r1["o"][:, 0], g["o"][[5], 1], atol=1e-12)


# --------------------------------------------------------------- plan pins (SPEC worked examples)

def test_spec_golden_examples():
    G = json.load(open(GOLDEN))
    for e in G["causal_pairs"]:
        assert oracle.causal_pairs(e["s_len"], e["prefix"]) == e["pairs"], e["cite"]
    for e in G["partition_equal"]:
        assert oracle.partition_equal(e["S"], e["N"]) == e["lengths"], e["cite"]
    for e in G["offload_alpha"]:
        assert oracle.offload_alpha(e["A"], e["m_threshold"]) == e["alpha"], e["cite"]
    for e in G["memory_timeline"]:
        assert oracle.memory_timeline(e["A"], e["alpha"]) == e["M"], e["cite"]


def test_pair_count_closed_form_and_brute_force():
    rng = np.random.default_rng(1)
    for _ in range(20):
        S = int(rng.integers(1, 200))
        N = int(rng.integers(1, min(S, 9) + 1))
        off = ragged_offsets(S, N, seed=int(rng.integers(1 << 30))) if N > 1 else [0, S]
        assert oracle.total_pairs(off) == S * (S + 1) // 2
        brute = sum(1 for p in range(S) for t in range(S) if t <= p)
        assert brute == S * (S + 1) // 2
    assert oracle.attention_flops(32, 128, [0, 131072], "fwd") == 4 * 128 * 32 * 131072 * 131073 // 2
    with pytest.raises(ValueError):
        oracle.partition_equal(3, 4)
    with pytest.raises(ValueError):
        oracle.causal_pairs(0, 0)
    assert oracle.offsets_from_lengths([3, 1, 2]) == [0, 3, 4, 6]
    assert oracle.offload_alpha([4, 2, 1], 2, last=0.0) == [0.5, 1.0, 0.0]
