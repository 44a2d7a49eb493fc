"""fp64 oracle for subsequence-chunked causal attention — TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py for the usage rule (tests / smoke / bench cpu_baseline only).

What the method computes:

  P:356 [§5.1 Two-Level Activation Management]: "due to the casual mask, after
  attention computation, Q_i will not be used in the forward pass anymore, while
  K_i and V_i need to participate in the following Q_N computation, where i<N".
  So chunk i's queries attend to the keys/values of chunks 0..i with a causal
  mask on absolute token positions.

Chunking plus online softmax (FlashAttention / blockwise attention, cited at
P:134 [§2.1] and P:594 [§8 Related Work]) is an exact algebraic rewrite of dense
causal softmax attention, so the reference result is the textbook definition
(L2: row p sees keys t <= p; L1: tau = 1/sqrt(d); L5: natural-log LSE):

    s_pt  = tau <q_p, k_t>            (t <= p)
    LSE_p = log sum_{t<=p} exp(s_pt)
    P_pt  = exp(s_pt - LSE_p)
    O_p   = sum_t P_pt v_t

and its gradients for the scalar L = sum <dO, O>:

    Delta_p = <dO_p, O_p>
    dV_t    = sum_{p>=t} P_pt dO_p
    dS_pt   = P_pt (<dO_p, v_t> - Delta_p)
    dQ_p    = tau sum_t dS_pt k_t
    dK_t    = tau sum_p dS_pt q_p

Layouts match the C ABI: q/k/v/o/do/dq/dk/dv are token-major ``[S, h, d]``;
lse and delta are head-major ``[h, S]``.  Everything is float64.
"""

from __future__ import annotations

import numpy as np


def _scale(d: int, scale: float | None) -> float:
    # Reading L1: the paper never states the softmax scale; use 1/sqrt(d).
    return 1.0 / np.sqrt(d) if (scale is None or scale == 0.0) else float(scale)


def _f64(*xs):
    return [np.asarray(x, dtype=np.float64) for x in xs]


# ----------------------------------------------------------------------------
# 1. Dense definition (brute force, S <= ~4096)
# ----------------------------------------------------------------------------

def causal_attention_dense(q, k, v, scale=None):
    """Dense causal softmax attention, the definition above.

    Returns (o [S,h,d], lse [h,S]).  Builds the full S x S score matrix per head.
    """
    q, k, v = _f64(q, k, v)
    S, h, d = q.shape
    tau = _scale(d, scale)
    o = np.empty_like(q)
    lse = np.empty((h, S))
    mask = np.tril(np.ones((S, S), dtype=bool))  # row p sees t <= p (L2)
    for hh in range(h):
        s = tau * (q[:, hh, :] @ k[:, hh, :].T)
        s = np.where(mask, s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        e = np.exp(s - m)
        l = e.sum(axis=1, keepdims=True)
        p = e / l
        o[:, hh, :] = p @ v[:, hh, :]
        lse[hh] = (m + np.log(l))[:, 0]
    return o, lse


def causal_attention_dense_bwd(q, k, v, do, scale=None):
    """Dense forward + backward of L = sum <dO, O> (formulas in module doc).

    Returns a dict with o, lse, delta, dq, dk, dv.
    """
    q, k, v, do = _f64(q, k, v, do)
    S, h, d = q.shape
    tau = _scale(d, scale)
    o, lse = causal_attention_dense(q, k, v, tau)
    mask = np.tril(np.ones((S, S), dtype=bool))
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    delta = np.einsum("shd,shd->hs", do, o)
    for hh in range(h):
        s = tau * (q[:, hh, :] @ k[:, hh, :].T)
        p = np.where(mask, np.exp(np.where(mask, s, 0.0) - lse[hh][:, None]), 0.0)
        dv[:, hh, :] = p.T @ do[:, hh, :]
        dp = do[:, hh, :] @ v[:, hh, :].T
        ds = p * (dp - delta[hh][:, None])
        dq[:, hh, :] = tau * (ds @ k[:, hh, :])
        dk[:, hh, :] = tau * (ds.T @ q[:, hh, :])
    return dict(o=o, lse=lse, delta=delta, dq=dq, dk=dk, dv=dv)


# ----------------------------------------------------------------------------
# 2. Chunked online-softmax forward, in the paper's chunk order
# ----------------------------------------------------------------------------

def empty_state(rows: int, h: int, d: int):
    """Identity of merge_states: acc = 0, m = -inf, l = 0 (reading L14/a2)."""
    return (np.zeros((rows, h, d)), np.full((h, rows), -np.inf), np.zeros((h, rows)))


def merge_states(a, b):
    """Merge two partial online-softmax states (acc unnormalised, m, l).

    (acc, m, l) over a key set T means: m_p = max_{t in T} s_pt,
    l_p = sum_{t in T} exp(s_pt - m_p), acc_p = sum_{t in T} exp(s_pt - m_p) v_t.
    The union of two disjoint key sets is obtained by rescaling both to the
    common max (FlashAttention's online softmax; blockwise merge).
    """
    acc_a, m_a, l_a = a
    acc_b, m_b, l_b = b
    m = np.maximum(m_a, m_b)
    # exp(-inf - (-inf)) is undefined: a side with m = -inf contributes nothing.
    with np.errstate(invalid="ignore"):
        fa = np.where(np.isneginf(m_a), 0.0, np.exp(m_a - np.where(np.isneginf(m), 0.0, m)))
        fb = np.where(np.isneginf(m_b), 0.0, np.exp(m_b - np.where(np.isneginf(m), 0.0, m)))
    l = fa * l_a + fb * l_b
    acc = acc_a * fa.T[:, :, None] + acc_b * fb.T[:, :, None]
    return acc, m, l


def finalize_state(state):
    """O = acc / l, LSE = m + ln l (reading L5: natural log)."""
    acc, m, l = state
    o = acc / l.T[:, :, None]
    lse = m + np.log(l)
    return o, lse


def _block_state(qi, kj, vj, tau, q_pos0, k_pos0):
    """Partial state of query rows qi (absolute positions q_pos0..) against one
    key block kj/vj (absolute positions k_pos0..), causal mask on absolute
    positions (reading L2)."""
    si, h, d = qi.shape
    sj = kj.shape[0]
    qpos = q_pos0 + np.arange(si)[:, None]
    kpos = k_pos0 + np.arange(sj)[None, :]
    visible = kpos <= qpos
    acc = np.zeros((si, h, d))
    m = np.full((h, si), -np.inf)
    l = np.zeros((h, si))
    for hh in range(h):
        s = tau * (qi[:, hh, :] @ kj[:, hh, :].T)
        s = np.where(visible, s, -np.inf)
        mh = s.max(axis=1)
        ok = ~np.isneginf(mh)
        e = np.zeros_like(s)
        e[ok] = np.exp(s[ok] - mh[ok][:, None])
        m[hh] = mh
        l[hh] = e.sum(axis=1)
        acc[:, hh, :] = e @ vj[:, hh, :]
    return acc, m, l


def chunked_attention_fwd(q, k, v, offsets, scale=None):
    """Chunked forward in the paper's order (SURVEY §8(c) oracle item 2).

    for i = 0..N-1 (ascending, "(i-1)-th ... overlapped with ... i-th"):
      for j = 0..i:      block = tau Q_i K_j^T (mask only bites when j = i)
                         m_new = max(m, rowmax(block)); l, acc rescaled by
                         exp(m - m_new) and the block's contribution added
      O_i = acc / l, LSE_i = m + ln l
    Returns (o [S,h,d], lse [h,S]) assembled over chunks.
    """
    q, k, v = _f64(q, k, v)
    S, h, d = q.shape
    tau = _scale(d, scale)
    offsets = [int(x) for x in offsets]
    o = np.empty_like(q)
    lse = np.empty((h, S))
    for i in range(len(offsets) - 1):
        ci, ce = offsets[i], offsets[i + 1]
        qi = q[ci:ce]
        acc, m, l = empty_state(ce - ci, h, d)
        for j in range(i + 1):
            cj, cje = offsets[j], offsets[j + 1]
            kj, vj = k[cj:cje], v[cj:cje]
            si, sj = ce - ci, cje - cj
            qpos = ci + np.arange(si)[:, None]
            kpos = cj + np.arange(sj)[None, :]
            visible = kpos <= qpos
            for hh in range(h):
                blk = tau * (qi[:, hh, :] @ kj[:, hh, :].T)
                blk = np.where(visible, blk, -np.inf)
                m_new = np.maximum(m[hh], blk.max(axis=1))
                alpha = np.where(np.isneginf(m[hh]), 0.0, np.exp(m[hh] - m_new))
                e = np.where(visible, np.exp(np.where(visible, blk, 0.0) - m_new[:, None]), 0.0)
                l[hh] = l[hh] * alpha + e.sum(axis=1)
                acc[:, hh, :] = acc[:, hh, :] * alpha[:, None] + e @ vj[:, hh, :]
                m[hh] = m_new
        o[ci:ce], lse[:, ci:ce] = finalize_state((acc, m, l))
    return o, lse


def chunked_attention_fwd_windows(q, k, v, offsets, windows, scale=None):
    """Forward where chunk i's prior-KV set 0..i is visited in caller-chosen
    windows (the ABI's FIRST/LAST carry).  ``windows[i]`` is a
    list of lists of chunk ids partitioning 0..i, in any order.  Each window's
    partial state is merged into the running state with merge_states.
    """
    q, k, v = _f64(q, k, v)
    S, h, d = q.shape
    tau = _scale(d, scale)
    offsets = [int(x) for x in offsets]
    o = np.empty_like(q)
    lse = np.empty((h, S))
    for i in range(len(offsets) - 1):
        ci, ce = offsets[i], offsets[i + 1]
        seen = sorted(j for w in windows[i] for j in w)
        if seen != list(range(i + 1)):
            raise ValueError(f"windows for chunk {i} must partition 0..{i}")
        state = empty_state(ce - ci, h, d)
        for w in windows[i]:
            for j in w:
                cj, cje = offsets[j], offsets[j + 1]
                part = _block_state(q[ci:ce], k[cj:cje], v[cj:cje], tau, ci, cj)
                state = merge_states(state, part)
        o[ci:ce], lse[:, ci:ce] = finalize_state(state)
    return o, lse


# ----------------------------------------------------------------------------
# 3. Chunked backward, reverse chunk order (L11)
# ----------------------------------------------------------------------------

def chunked_attention_bwd(q, k, v, o, lse, do, offsets, scale=None):
    """Backward of chunked attention, chunks i = N-1..0 (reading L11).

    Per chunk i: Delta_i = rowsum(dO_i * O_i); for j = 0..i:
      P = exp(tau Q_i K_j^T - LSE_i) (masked to 0), dV_j += P^T dO_i,
      dP = dO_i V_j^T, dS = P * (dP - Delta_i), dQ_i += tau dS K_j,
      dK_j += tau dS^T Q_i.
    dK_j / dV_j are final once chunk j has been processed.
    Returns dict(dq, dk, dv, delta).
    """
    q, k, v, o, lse, do = _f64(q, k, v, o, lse, do)
    S, h, d = q.shape
    tau = _scale(d, scale)
    offsets = [int(x) for x in offsets]
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    delta = np.einsum("shd,shd->hs", do, o)
    N = len(offsets) - 1
    for i in range(N - 1, -1, -1):
        ci, ce = offsets[i], offsets[i + 1]
        for j in range(i + 1):
            cj, cje = offsets[j], offsets[j + 1]
            qpos = ci + np.arange(ce - ci)[:, None]
            kpos = cj + np.arange(cje - cj)[None, :]
            visible = kpos <= qpos
            for hh in range(h):
                s = tau * (q[ci:ce, hh, :] @ k[cj:cje, hh, :].T)
                p = np.where(visible, np.exp(np.where(visible, s, 0.0) - lse[hh, ci:ce][:, None]), 0.0)
                dv[cj:cje, hh, :] += p.T @ do[ci:ce, hh, :]
                dp = do[ci:ce, hh, :] @ v[cj:cje, hh, :].T
                ds = p * (dp - delta[hh, ci:ce][:, None])
                dq[ci:ce, hh, :] += tau * (ds @ k[cj:cje, hh, :])
                dk[cj:cje, hh, :] += tau * (ds.T @ q[ci:ce, hh, :])
    return dict(dq=dq, dk=dk, dv=dv, delta=delta)


# ----------------------------------------------------------------------------
# 4. Sampled outputs at sizes where the full oracle cannot run
# ----------------------------------------------------------------------------

def _rows_block(qh, kh, vh, doh, rows, tau):
    """Exact per-row quantities for one head: o, lse, delta, dq (each row uses
    only keys t <= p; O(p d) work per row)."""
    R = len(rows)
    d = qh.shape[1]
    o = np.empty((R, d))
    lse = np.empty(R)
    delta = np.empty(R)
    dq = np.empty((R, d))
    for n, p in enumerate(rows):
        s = tau * (kh[: p + 1] @ qh[p])
        m = s.max()
        e = np.exp(s - m)
        l = e.sum()
        pr = e / l
        o[n] = pr @ vh[: p + 1]
        lse[n] = m + np.log(l)
        if doh is not None:
            delta[n] = doh[p] @ o[n]
            dp = vh[: p + 1] @ doh[p]
            ds = pr * (dp - delta[n])
            dq[n] = tau * (ds @ kh[: p + 1])
    return o, lse, delta, dq


def sampled_rows(q, k, v, rows, do=None, heads=None, scale=None):
    """O_p, LSE_p (and Delta_p, dQ_p when dO given) for selected query rows,
    computed from the definition row by row.  q/k/v/do may be any array-likes
    indexable as [S, h, d] (rows beyond max(rows) are never touched).
    Returns dict(o [R,H,d], lse [H,R], delta [H,R], dq [R,H,d]) for heads H.
    """
    rows = [int(r) for r in rows]
    pmax = max(rows) + 1
    d = q.shape[2]
    tau = _scale(d, scale)
    heads = list(range(q.shape[1])) if heads is None else list(heads)
    H, R = len(heads), len(rows)
    out = dict(o=np.empty((R, H, d)), lse=np.empty((H, R)), delta=np.empty((H, R)), dq=np.empty((R, H, d)))
    for n, hh in enumerate(heads):
        qh = np.asarray(q[:pmax, hh, :], dtype=np.float64)
        kh = np.asarray(k[:pmax, hh, :], dtype=np.float64)
        vh = np.asarray(v[:pmax, hh, :], dtype=np.float64)
        doh = None if do is None else np.asarray(do[:pmax, hh, :], dtype=np.float64)
        o, lse, delta, dq = _rows_block(qh, kh, vh, doh, rows, tau)
        out["o"][:, n], out["lse"][n], out["delta"][n], out["dq"][:, n] = o, lse, delta, dq
    return out


def sampled_key_grads(q, k, v, do, keys, heads=None, scale=None, row_block=256):
    """dK_t, dV_t for selected keys t, from the definition:
        dV_t = sum_{p >= t} P_pt dO_p,   dK_t = tau sum_{p >= t} dS_pt q_p,
        dS_pt = P_pt (<dO_p, v_t> - Delta_p),  Delta_p = <dO_p, O_p>,
    where every row p >= min(keys) gets its exact P row, LSE_p and O_p from its
    own full causal prefix (keys 0..p).  Rows are taken in blocks of
    ``row_block``; a block [r0, r1) only needs keys < r1 (causality), and only
    its diagonal square needs the t > p mask.
    Cost O((S - min(keys)) * S * d) per head, so pick keys near the end unless
    the time is affordable.  Returns dict(dk [K,H,d], dv [K,H,d]).
    """
    keys = np.asarray([int(t) for t in keys])
    S, _, d = q.shape
    tau = _scale(d, scale)
    heads = list(range(q.shape[1])) if heads is None else list(heads)
    t0 = int(keys.min())
    dk = np.zeros((len(keys), len(heads), d))
    dv = np.zeros((len(keys), len(heads), d))
    for n, hh in enumerate(heads):
        qh = np.asarray(q[:, hh, :], dtype=np.float64)
        kh = np.asarray(k[:, hh, :], dtype=np.float64)
        vh = np.asarray(v[:, hh, :], dtype=np.float64)
        doh = np.asarray(do[:, hh, :], dtype=np.float64)
        vk = vh[keys]
        for r0 in range(t0, S, row_block):
            r1 = min(S, r0 + row_block)
            s = tau * (qh[r0:r1] @ kh[:r1].T)                       # rows r0..r1-1, keys 0..r1-1
            diag = s[:, r0:r1]
            diag[np.triu_indices(r1 - r0, 1)] = -np.inf              # t > p masked
            m = s.max(axis=1, keepdims=True)
            np.subtract(s, m, out=s)
            np.exp(s, out=s)
            l = s.sum(axis=1, keepdims=True)
            np.divide(s, l, out=s)                                   # s now holds the exact P rows
            o = s @ vh[:r1]
            delta = np.einsum("rd,rd->r", doh[r0:r1], o)
            pk = np.zeros((r1 - r0, len(keys)))
            vis = keys < r1                                          # keys no row of the block sees: P = 0
            pk[:, vis] = s[:, keys[vis]]
            dpk = doh[r0:r1] @ vk.T                                  # [rows, K]
            dsk = pk * (dpk - delta[:, None])
            dv[:, n] += pk.T @ doh[r0:r1]
            dk[:, n] += tau * (dsk.T @ qh[r0:r1])
    return dict(dk=dk, dv=dv)


# ----------------------------------------------------------------------------
# 5. Finite differences
# ----------------------------------------------------------------------------

def fd_grad(f, x, eps=1e-6):
    """Central finite differences of scalar f at x (fp64): (f(x+e) - f(x-e))/2e."""
    x = np.array(x, dtype=np.float64, copy=True)
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        idx = it.multi_index
        old = x[idx]
        x[idx] = old + eps
        fp = f(x)
        x[idx] = old - eps
        fm = f(x)
        x[idx] = old
        g[idx] = (fp - fm) / (2 * eps)
    return g
