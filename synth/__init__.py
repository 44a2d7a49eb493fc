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


# ---------------------------------------------------------------- full layer
# Parameter shapes of one GPT layer (hidden H, nn.Linear [out, in] layout); the
# order matches oracle.layer.PARAM_NAMES.  Recipe:
# GPT/Megatron initialisation — weights N(0, 0.02), the two projections that
# feed the residual stream (w_o, w_2) N(0, 0.02/sqrt(2 L)) with L = 32 layers,
# biases N(0, 0.02), LayerNorm gamma 1 + N(0, 0.1), beta N(0, 0.1); the layer
# input x and the upstream gradient dz are N(0, 1).  Values are rounded to bf16
# for bf16 runs.
LAYER_PARAMS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")


def layer_param_shapes(H: int):
    return {"ln1_g": (H,), "ln1_b": (H,), "w_qkv": (3 * H, H), "b_qkv": (3 * H,), "w_o": (H, H), "b_o": (H,),
            "ln2_g": (H,), "ln2_b": (H,), "w_1": (4 * H, H), "b_1": (4 * H,), "w_2": (H, 4 * H), "b_2": (H,)}


def make_layer_params(H: int, seed: int = 0, dtype=torch.bfloat16, device="cpu", n_layers: int = 32):
    out = {}
    g = torch.Generator(device=device)
    resid_std = 0.02 / (2.0 * n_layers) ** 0.5
    for n, (name, shape) in enumerate(layer_param_shapes(H).items()):
        g.manual_seed(int(seed) * 1_000_003 + 7_000_001 + n)
        x = torch.randn(shape, generator=g, dtype=torch.float32, device=device)
        if name in ("ln1_g", "ln2_g"):
            x = 1.0 + 0.1 * x
        elif name in ("ln1_b", "ln2_b"):
            x = 0.1 * x
        elif name in ("w_o", "w_2"):
            x = resid_std * x
        else:
            x = 0.02 * x
        out[name] = x.to(dtype)
    return out


def make_layer_io(S: int, H: int, seed: int = 0, dtype=torch.bfloat16, device="cpu"):
    """dict(x, dz) of [S, H] tensors, N(0, 1)."""
    out = {}
    for n, name in enumerate(("x", "dz")):
        g = torch.Generator(device=device)
        g.manual_seed(int(seed) * 1_000_003 + 9_000_001 + n)
        out[name] = torch.randn((S, H), generator=g, dtype=torch.float32, device=device).to(dtype)
    return out
