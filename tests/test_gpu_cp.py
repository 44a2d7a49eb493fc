"""Context-parallel ring attention on the bf16 tcgen05 kernels:
2 ranks sharing one B200 (gloo, host-staged ring hops — the only GPU count this
environment has; NCCL would refuse two ranks on one device).  Each rank holds its
zigzag chunks; O, LSE, dQ, dK, dV of its own tokens are compared with the dense
oracle element by element."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth import make_inputs

pytestmark = pytest.mark.gpu

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, h, N, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_10377_b200 import cp, sppo
    torch.cuda.set_device(0)
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    L = sppo.Layout(h, 128, off)
    x = make_inputs(S, range(h), 128, seed=41, dtype=torch.bfloat16)
    own = cp.owned_chunks(N, world, rank)
    rows = torch.cat([torch.arange(off[i], off[i + 1]) for i in own])
    loc = {t: x[t][rows].contiguous().cuda() for t in ("q", "k", "v", "do")}
    ra = cp.RingAttention(ctx, L)
    ra.forward(loc["q"], loc["k"], loc["v"])
    ra.backward(loc["q"], loc["k"], loc["v"], loc["do"])
    torch.cuda.synchronize()
    ctx.sync()
    lse = torch.cat([ra._lse(i).view(h, -1) for i in own], dim=1)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), rows=rows.numpy(), o=ra.o.float().cpu().numpy(),
             lse=lse.cpu().numpy(), dq=ra.dq.float().cpu().numpy(), dk=ra.dk.float().cpu().numpy(),
             dv=ra.dv.float().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


@pytest.mark.parametrize("S,h,N", [(2048, 2, 4), (1500, 1, 8)])
def test_ring_two_ranks_matches_oracle(tmp_path, S, h, N):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), S, h, N, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x = make_inputs(S, range(h), 128, seed=41, dtype=torch.bfloat16)
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref = oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])
    covered = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        rows = d["rows"]
        covered += list(rows)
        np.testing.assert_allclose(d["o"], ref["o"][rows], **O_TOL)
        np.testing.assert_allclose(d["lse"], ref["lse"][:, rows], atol=1e-3, rtol=0)
        for key in ("dq", "dk", "dv"):
            np.testing.assert_allclose(d[key], ref[key][rows], **G_TOL, err_msg=f"rank {r} {key}")
    assert sorted(covered) == list(range(S))


def test_finalize_cast_and_errors():
    """sppo_finalize (a7): RNE fp32 -> bf16 cast / fp32 copy; n % 4 and alignment checked."""
    from paper_2503_10377_b200 import sppo
    ctx = sppo.Context(0)
    src = torch.randn(4096, device="cuda") * 3
    dst = torch.empty(4096, dtype=torch.bfloat16, device="cuda")
    ctx.finalize(src, dst, sppo.SPPO_BF16)
    torch.cuda.synchronize()
    assert torch.equal(dst, src.to(torch.bfloat16))
    d32 = torch.empty(4096, device="cuda")
    ctx.finalize(src, d32, sppo.SPPO_FP32)
    torch.cuda.synchronize()
    assert torch.equal(d32, src)
    with pytest.raises(sppo.SppoError) as e:
        ctx.finalize(src[:6], dst[:6], sppo.SPPO_BF16)
    assert e.value.name == "SPPO_E_SHAPE"
    with pytest.raises(sppo.SppoError) as e:
        ctx.finalize(src[1:5], dst[:4], sppo.SPPO_BF16)
    assert e.value.name == "SPPO_E_ALIGN"
    ctx.close()
