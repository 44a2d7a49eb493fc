"""Host-side formulas of the hot path, fp64/integer — TEST INFRASTRUCTURE ONLY.

(See oracle/__init__.py for the usage rule.)

  * causal pair count of a chunk   — S:43-50 [cost_model.forward_flops, c_lin = 0];
    P:256 [§3.2] "the computational load for later token positions ... is heavier".
  * FLOP convention                — BASELINE.md: fwd 4d per causal (q,k) pair,
    bwd 10d per pair (2.5x fwd incl. the QK^T recompute).
  * equal partition                — P:253 [§3.2] "length-based policy";
    S:112-120 [partitioner.partition_equal], remainder to the first chunks.
  * offload ratio alpha            — P:371-377 [§5.2] "alpha_i * A_i = M_threshold";
    S:238-246 [offload_planner.compute_offload_ratios]; reading L9 for the last chunk.
  * memory recurrence              — P:373 [§5.2] M_i = M_{i-1} + A_i - alpha_{i-1} A_{i-1};
    S:247-254 [offload_planner.memory_timeline].
"""

from __future__ import annotations


def causal_pairs(s_len: int, prefix: int) -> int:
    """Causal (q,k) pairs of a chunk of s_len rows whose first row sits after
    ``prefix`` earlier tokens: sum_{t=1}^{s_len} (prefix + t)."""
    if s_len < 1 or prefix < 0:
        raise ValueError("s_len >= 1 and prefix >= 0 required")
    return sum(prefix + t for t in range(1, s_len + 1))


def total_pairs(offsets) -> int:
    """Sum over chunks of causal_pairs(s_i, c_i)."""
    offsets = [int(x) for x in offsets]
    return sum(causal_pairs(offsets[i + 1] - offsets[i], offsets[i]) for i in range(len(offsets) - 1))


def attention_flops(heads: int, head_dim: int, offsets, part: str = "fwd+bwd") -> int:
    """Algorithmic FLOPs: 4 d per pair (QK^T + PV) forward, 10 d per pair
    backward (QK^T recompute, dV, dP, dQ, dK), per head."""
    per_pair = {"fwd": 4, "bwd": 10, "fwd+bwd": 14}[part] * head_dim
    return heads * per_pair * total_pairs(offsets)


def partition_equal(S: int, N: int):
    """Chunk lengths differing by at most 1, the first S mod N chunks one longer
    (S:116-119).  Returns the list of lengths."""
    if not (1 <= N <= S):
        raise ValueError("1 <= N <= S required")
    base, rem = divmod(S, N)
    return [base + (1 if i < rem else 0) for i in range(N)]


def partition_min_max_pairs(S: int, N: int, lin: int = 0):
    """FLOPs-balanced partition (P:253, P:256, P:327 [§3.2, §4]):
    the N chunk lengths minimising max_i causal_pairs(s_i, c_i), by exact dynamic
    programming over split points (small S only).  Among optimal partitions the
    lexicographically largest length vector is returned ("ties broken toward the
    longer first chunk").  Cost of a chunk [a, b) is T(b) - T(a) with
    T(x) = x (x + 1) / 2 (the causal pairs of rows a..b-1), plus lin (b - a) for a
    per-token linear term (c_lin: the token-wise work of a full layer)."""
    if not (1 <= N <= S):
        raise ValueError("1 <= N <= S required")
    T0 = lambda x: x * (x + 1) // 2  # noqa: E731
    T = lambda x: T0(x) + lin * x  # noqa: E731  (cost(a, b) = T(b) - T(a))
    INF = float("inf")
    # best[k][e] = min over partitions of [0, e) into k chunks of the max chunk cost
    best = [[INF] * (S + 1) for _ in range(N + 1)]
    best[0][0] = 0
    for k in range(1, N + 1):
        for e in range(k, S + 1):
            best[k][e] = min(max(best[k - 1][a], T(e) - T(a)) for a in range(k - 1, e))
    opt = best[N][S]
    # reconstruct the lexicographically largest lengths achieving opt: walk forward,
    # taking each chunk as long as possible while the rest stays feasible.
    # feasible(k, a) := the suffix [a, S) splits into k chunks each of cost <= opt
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def feasible(k, a):
        if k == 0:
            return a == S
        return any(T(b) - T(a) <= opt and feasible(k - 1, b) for b in range(a + 1, S - k + 2))

    lengths, a = [], 0
    for k in range(N, 0, -1):
        b = max(b for b in range(a + 1, S - k + 2) if T(b) - T(a) <= opt and feasible(k - 1, b))
        lengths.append(b - a)
        a = b
    return lengths


def offsets_from_lengths(lengths):
    """c_0 = 0, c_{i+1} = c_i + s_i."""
    out = [0]
    for s in lengths:
        if s < 1:
            raise ValueError("chunk lengths must be >= 1")
        out.append(out[-1] + int(s))
    return out


def offload_alpha(A, m_threshold, last: float = 1.0):
    """alpha_i = min(1, M_threshold / A_i) for i < last chunk;
    A_i = 0 gives alpha_i = 1 (nothing to offload).  The last chunk's
    ratio is ``last``: 1.0 per the paper ("alpha_k = 1 for final
    subsequence"), 0.0 in the single-layer bench (reading L9: its backward
    consumes it immediately).  ``m_threshold`` is the paper's constant
    M_threshold, or a per-chunk list M_i = BW_D2H * T_comp(i+1) (reading L9,
    "sequence-aware": the offload of i overlaps the compute of i+1)."""
    n = len(A)
    thr = list(m_threshold) if hasattr(m_threshold, "__len__") else [m_threshold] * n
    out = []
    for i, a in enumerate(A):
        if i == n - 1:
            out.append(float(last))
        elif a <= 0:
            out.append(1.0)
        else:
            out.append(min(1.0, float(thr[i]) / float(a)))
    return out


def memory_timeline(A, alpha):
    """M_i = M_{i-1} + A_i - alpha_{i-1} A_{i-1}, M_{-1} = 0."""
    if len(A) != len(alpha):
        raise ValueError("length mismatch")
    M = []
    prev = 0.0
    for i, a in enumerate(A):
        shed = alpha[i - 1] * A[i - 1] if i > 0 else 0.0
        prev = prev + a - shed
        M.append(prev)
    return M


# ---------------------------------------------------------------- subsequence pipeline
def bubble_ratio(p: int, N: int) -> float:
    """P:282-285 [§3.3 "Inevitable bubble overhead"]: t_b = (p-1) F(N)/N,
    R_b = (p-1)/N, T = (p-1+N)/N F(N)."""
    return (p - 1) / N


def pipeline_makespan(p: int, N: int, t_fwd, t_bwd):
    """Event-driven simulation of the subsequence pipeline: p stages, N chunks;
    stage s runs fwd(0..N-1) in order, each after stage s-1's fwd of that chunk;
    then bwd(N-1..0) in order, each after stage s+1's bwd of that chunk (the
    last stage starts its backward after its own last forward).  Task times are
    scalars (uniform) or per-chunk lists.  Returns (makespan, per-stage list of
    (kind, chunk, start, end))."""
    tf = list(t_fwd) if hasattr(t_fwd, "__len__") else [t_fwd] * N
    tb = list(t_bwd) if hasattr(t_bwd, "__len__") else [t_bwd] * N
    fend = [[0.0] * N for _ in range(p)]
    bend = [[0.0] * N for _ in range(p)]
    log = [[] for _ in range(p)]
    for s in range(p):
        t = 0.0
        for i in range(N):
            start = max(t, fend[s - 1][i] if s > 0 else 0.0)
            t = start + tf[i]
            fend[s][i] = t
            log[s].append(("fwd", i, start, t))
    for s in range(p - 1, -1, -1):
        t = fend[s][N - 1]
        for i in range(N - 1, -1, -1):
            start = max(t, bend[s + 1][i] if s + 1 < p else 0.0)
            t = start + tb[i]
            bend[s][i] = t
            log[s].append(("bwd", i, start, t))
    return max(bend[s][0] for s in range(p)), log


def msp_phases(PP: int, N: int, stage: int):
    """Multiplexed sequence partitioning (P:420-455 [§6.2]) for pipeline stage
    `stage`: subsequence ids of the Left-SP, Steady and Right-SP phases and the
    GPU (stage) ranges that run the two SP phases.

    The Definition's inclusive bounds overlap (Left {0..PP-1-i} and Steady
    {PP-1-i..N-i} share PP-1-i; Steady reaches N-i, which is Right's first id and
    equals N for i = 0).  Reading L18: the paper's worked example (Table
    "multiplexed sequence partitioning for PP=4, N=8") decides:
        Left = {0 .. PP-2-i},  Steady = {PP-1-i .. N-1-i},  Right = {N-i .. N-1}
    and the SP ranges follow the Communication-Scope definition
        Left-SP range = {i .. PP-1}  (empty when Left is empty),
        Right-SP range = {0 .. i}    (empty when Right is empty)."""
    if not (1 <= PP and PP <= N and 0 <= stage < PP):
        raise ValueError("need 1 <= PP <= N and 0 <= stage < PP")
    left = list(range(0, PP - 1 - stage))
    steady = list(range(PP - 1 - stage, N - stage))
    right = list(range(N - stage, N))
    left_sp = list(range(stage, PP)) if left else []
    right_sp = list(range(0, stage + 1)) if right else []
    return dict(left=left, steady=steady, right=right, left_sp=left_sp, right_sp=right_sp)
