"""Host-side logic of the per-chunk layer that needs no GPU: the tensor-parallel
parameter sharding (Megatron layout) reassembles the full parameters, and the
row-/column-parallel split of the layer's linear maps sums to the full product
(checked with fp64 torch on the CPU, the oracle's layer definition)."""

import torch

import synth
from paper_2503_10377_b200.engine_layer import shard_params


def test_shards_reassemble_the_full_parameters():
    H, heads = 256, 4
    full = synth.make_layer_params(H, 3, dtype=torch.float64)
    for size in (1, 2, 4):
        sh = [shard_params(full, H, heads, r, size) for r in range(size)]
        Hl = H // size
        for k in range(3):  # q, k, v blocks of W_qkv: this rank's heads of each
            blk = torch.cat([s["w_qkv"][k * Hl:(k + 1) * Hl] for s in sh])
            assert torch.equal(blk, full["w_qkv"][k * H:(k + 1) * H])
        assert torch.equal(torch.cat([s["w_o"] for s in sh], dim=1), full["w_o"])
        assert torch.equal(torch.cat([s["w_1"] for s in sh]), full["w_1"])
        assert torch.equal(torch.cat([s["b_1"] for s in sh]), full["b_1"])
        assert torch.equal(torch.cat([s["w_2"] for s in sh], dim=1), full["w_2"])
        for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2"):
            assert all(s[k] is full[k] for s in sh)


def test_row_parallel_partials_sum_to_the_full_projection():
    """out-proj / fc2 are row-parallel: sum_r o_r W_o[:, r]^T == o W_o^T (the
    all-reduce of the partial sums), and column-parallel fc1 concatenates."""
    H, heads, size, S = 128, 4, 4, 16
    full = synth.make_layer_params(H, 5, dtype=torch.float64)
    g = torch.Generator().manual_seed(0)
    o = torch.randn(S, H, generator=g, dtype=torch.float64)
    b = torch.randn(S, H, generator=g, dtype=torch.float64)
    sh = [shard_params(full, H, heads, r, size) for r in range(size)]
    Hl = H // size
    part = sum(o[:, r * Hl:(r + 1) * Hl] @ sh[r]["w_o"].T for r in range(size))
    torch.testing.assert_close(part, o @ full["w_o"].T, rtol=1e-12, atol=1e-12)
    cols = torch.cat([b @ s["w_1"].T for s in sh], dim=1)
    torch.testing.assert_close(cols, b @ full["w_1"].T, rtol=1e-12, atol=1e-12)
