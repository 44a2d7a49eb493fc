"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method — only random-number generation
and dtype rounding of the generated values — so that both sides consume the
exact same data:

  * Q, K, V, dO are iid N(0, 1) fp32, generated per GLOBAL head index with its
    own seed, so a head-sharded run (rank g owns heads [g*h/G, (g+1)*h/G)) sees
    bit-identical per-head data to an unsharded run (SURVEY §8(c) "Inputs").
  * For bf16 runs the fp32 draws are rounded to bf16 (round-to-nearest-even);
    the oracle up-casts those bf16 values to fp64.
  * Shapes follow the paper's workloads: GPT-7B/13B/65B attention, d = 128,
    h = 32 / 40 / 64, token-major [S, h, d].
"""

from __future__ import annotations

import torch

_TENSORS = ("q", "k", "v", "do")


def head_seed(seed: int, tensor: str, head: int) -> int:
    """Counter-style seed for (tensor, global head)."""
    return int(seed) * 1_000_003 + _TENSORS.index(tensor) * 100_003 + int(head)


def make_tensor(tensor: str, S: int, heads, d: int, seed: int = 0, dtype=torch.bfloat16,
                device="cpu") -> torch.Tensor:
    """One of q/k/v/do as [S, len(heads), d] in ``dtype`` on ``device``.

    ``heads`` is an iterable of GLOBAL head indices.  Values are drawn per head
    with torch's generator for ``device`` (CPU Mersenne / CUDA Philox), so CPU-
    and GPU-generated tensors differ; each test picks one side to generate on
    and copies (never recomputes) to the other.
    """
    heads = list(heads)
    out = torch.empty((S, len(heads), d), dtype=dtype, device=device)
    g = torch.Generator(device=device)
    for n, hh in enumerate(heads):
        g.manual_seed(head_seed(seed, tensor, hh))
        x = torch.randn((S, d), generator=g, dtype=torch.float32, device=device)
        out[:, n, :] = x.to(dtype)
    return out


def make_inputs(S: int, heads, d: int, seed: int = 0, dtype=torch.bfloat16, device="cpu"):
    """dict(q, k, v, do) of [S, h, d] tensors (see make_tensor)."""
    return {t: make_tensor(t, S, heads, d, seed, dtype, device) for t in _TENSORS}


def ragged_offsets(S: int, N: int, seed: int = 0):
    """Random strictly increasing boundaries (odd, non-tile-multiple lengths) for
    edge-case parity tests."""
    g = torch.Generator().manual_seed(seed)
    cuts = torch.randperm(S - 1, generator=g)[: N - 1] + 1
    return [0] + sorted(int(c) for c in cuts) + [S]
