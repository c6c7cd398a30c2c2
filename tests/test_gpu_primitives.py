"""GPU self-tests of the tcgen05 building blocks (descriptor encodings)."""
import ctypes
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SELFTEST = os.path.join(ROOT, "paper_2311_05908_b200", "libfftconv_selftest.so")


@pytest.mark.gpu
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("N,K", [(16, 16), (128, 64), (256, 32), (64, 128)])
def test_tcgen05_mma_descriptors(a_mn, b_mn, N, K):
    import torch
    lib = ctypes.CDLL(SELFTEST)
    M = 128
    g = torch.Generator().manual_seed(N * 1000 + K + 10 * a_mn + b_mn)
    A = torch.randn(M, K, generator=g).half()
    B = torch.randn(K, N, generator=g).half()
    dA, dB = A.cuda(), B.cuda()
    dD = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    rc = lib.fcst_mma(ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                      ctypes.c_void_p(dD.data_ptr()), M, N, K, a_mn, b_mn)
    assert rc == 0
    ref = A.double() @ B.double()
    err = (dD.cpu().double() - ref).abs().max().item()
    assert err < 1e-3 * K, err
