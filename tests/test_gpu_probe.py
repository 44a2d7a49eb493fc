"""GPU probe of the tcgen05/TMEM/TMA building blocks (tests/cuda/tc_probe.cu):
one 128 x N x 128 BF16 product per mode, compared with a torch fp32 matmul of
the same bf16 values.  Pins the operand layouts the attention kernels rely on:
  mode 0  S = Q K^T      (A, B K-major in smem)
  mode 1  O = P V        (B MN-major in smem)
  mode 2  O = P V        (A from TMEM as packed bf16 pairs)
  mode 3  dQ = dS K      (A MN-major: dS stored transposed)
each with manual SW128 staging and with TMA SW128 loads."""

import ctypes
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(__file__), "cuda", "libtcprobe.so")


@pytest.mark.parametrize("use_tma", [0, 1])
@pytest.mark.parametrize("N", [128, 64])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_probe(mode, N, use_tma):
    lib = ctypes.CDLL(LIB)
    g = torch.Generator().manual_seed(mode * 10 + N + use_tma)
    A = torch.randn(128, 128, generator=g).to(torch.bfloat16)
    if mode == 0:
        B = torch.randn(N, 128, generator=g).to(torch.bfloat16)
        ref = A.float() @ B.float().T
    elif mode == 3:
        B = torch.randn(128, N, generator=g).to(torch.bfloat16)
        ref = A.float().T @ B.float()  # A holds At [k][m]
    else:
        B = torch.randn(128, N, generator=g).to(torch.bfloat16)
        ref = A.float() @ B.float()
    dA, dB = A.cuda(), B.cuda()
    D = torch.zeros(128, N, device="cuda")
    rc = lib.tc_probe_run(mode, N, use_tma, ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                          ctypes.c_void_p(D.data_ptr()))
    assert rc == 0, rc
    torch.testing.assert_close(D.cpu(), ref, atol=1e-3, rtol=1e-3)
