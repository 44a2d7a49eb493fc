"""FLOPs-balanced partition:
the oracle's exact DP is pinned by brute-force enumeration and the SPEC's worked
examples; the product's C implementation (sppo_partition_balanced) must equal
the oracle everywhere it can run."""

import itertools
import json
import os

import pytest

import oracle
from paper_2503_10377_b200 import sppo

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
T = lambda x: x * (x + 1) // 2


def brute(S, N):
    best = None
    for cuts in itertools.combinations(range(1, S), N - 1):
        o = [0, *cuts, S]
        L = [o[i + 1] - o[i] for i in range(N)]
        key = (max(T(o[i + 1]) - T(o[i]) for i in range(N)), [-x for x in L])
        if best is None or key < best[0]:
            best = (key, L)
    return best[1]


def test_oracle_dp_equals_brute_force():
    for S in range(1, 13):
        for N in range(1, S + 1):
            assert oracle.partition_min_max_pairs(S, N) == brute(S, N), (S, N)


def test_golden_spec_examples():
    for e in json.load(open(GOLDEN))["partition_balanced"]:
        assert oracle.partition_min_max_pairs(e["S"], e["N"]) == e["lengths"], e["cite"]
        off = sppo.partition_balanced(e["S"], e["N"])
        assert [off[i + 1] - off[i] for i in range(e["N"])] == e["lengths"], e["cite"]


@pytest.mark.parametrize("S,N", [(S, N) for S in range(1, 15) for N in range(1, S + 1)] +
                         [(200, 7), (1024, 4), (777, 5), (300, 300)])
def test_product_equals_oracle(S, N):
    assert sppo.partition_balanced(S, N) == oracle.offsets_from_lengths(oracle.partition_min_max_pairs(S, N))


def test_large_balanced_properties():
    """At bench sizes: lengths non-increasing ("longer subsequences first"),
    max chunk cost within one row's cost of the average (near-perfect balance)."""
    for S, N in ((131072, 16), (1048576, 64), (524288, 32)):
        off = sppo.partition_balanced(S, N)
        L = [off[i + 1] - off[i] for i in range(N)]
        assert sum(L) == S and all(a >= b for a, b in zip(L, L[1:]))
        cost = [T(off[i + 1]) - T(off[i]) for i in range(N)]
        assert max(cost) - T(S) / N <= S
    with pytest.raises(sppo.SppoError):
        sppo.partition_balanced(3, 4)


def brute_lin(S, N, lin):
    best = None
    for cuts in itertools.combinations(range(1, S), N - 1):
        o = [0, *cuts, S]
        L = [o[i + 1] - o[i] for i in range(N)]
        key = (max(T(o[i + 1]) - T(o[i]) + lin * L[i] for i in range(N)), [-x for x in L])
        if best is None or key < best[0]:
            best = (key, L)
    return best[1]


@pytest.mark.parametrize("lin", [1, 3, 10, 100])
def test_linear_term_partition_oracle_brute_and_product(lin):
    """S:46 forward_flops with c_lin > 0: chunk cost = pairs + lin * s (a full layer's
    token-wise work); DP oracle == brute force, product == oracle."""
    for S in range(1, 11):
        for N in range(1, S + 1):
            ref = brute_lin(S, N, lin)
            assert oracle.partition_min_max_pairs(S, N, lin) == ref, (S, N, lin)
            assert sppo.partition_balanced(S, N, lin) == oracle.offsets_from_lengths(ref), (S, N, lin)
    for S, N in ((200, 7), (777, 5)):
        assert sppo.partition_balanced(S, N, lin) == \
            oracle.offsets_from_lengths(oracle.partition_min_max_pairs(S, N, lin))


def test_linear_term_limits():
    """lin -> large: the token-wise term dominates and chunks approach equal lengths;
    lin = 0 is the attention-only partition."""
    S, N = 131072, 16
    assert sppo.partition_balanced(S, N, 0) == sppo.partition_balanced(S, N)
    off = sppo.partition_balanced(S, N, 1 << 30)
    L = [off[i + 1] - off[i] for i in range(N)]
    assert max(L) - min(L) <= 16
    off = sppo.partition_balanced(S, N, 36 * 4096 // 7)  # GPT-7B layer, fwd+bwd FLOPs
    L = [off[i + 1] - off[i] for i in range(N)]
    att = sppo.partition_balanced(S, N)
    assert all(a >= b for a, b in zip(L, L[1:])) and L[0] < att[1]  # less skewed than attention-only
