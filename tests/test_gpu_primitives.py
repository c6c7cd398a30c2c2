"""GPU self-tests of the tcgen05 building blocks (descriptor encodings, the
A-in-TMEM form and the M = 64 accumulator lane layout)."""
import ctypes
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SELFTEST = os.path.join(ROOT, "paper_2311_05908_b200", "libfftconv_selftest.so")


def _run(M, N, K, a_mn, b_mn, a_tmem=0, d_lane=0):
    import torch
    lib = ctypes.CDLL(SELFTEST)
    g = torch.Generator().manual_seed(N * 1000 + K + 10 * a_mn + b_mn + 7 * a_tmem + d_lane + M)
    A = torch.randn(M, K, generator=g).half()
    B = torch.randn(K, N, generator=g).half()
    dA, dB = A.cuda(), B.cuda()
    dD = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    rc = lib.fcst_mma(ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                      ctypes.c_void_p(dD.data_ptr()), M, N, K, a_mn, b_mn, a_tmem, d_lane)
    assert rc == 0
    ref = A.double() @ B.double()
    err = (dD.cpu().double() - ref).abs().max().item()
    assert err < 1e-3 * K, err


@pytest.mark.gpu
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("N,K", [(16, 16), (128, 64), (256, 32), (64, 128)])
def test_tcgen05_mma_descriptors(a_mn, b_mn, N, K):
    _run(128, N, K, a_mn, b_mn)


@pytest.mark.gpu
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("N,K", [(96, 64), (64, 128), (192, 32)])
def test_tcgen05_mma_a_in_tmem(b_mn, N, K):
    _run(128, N, K, 0, b_mn, a_tmem=1)


@pytest.mark.gpu
@pytest.mark.parametrize("d_lane", [0, 16])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("N,K", [(64, 128), (32, 64)])
def test_tcgen05_mma_m64_lanes(d_lane, a_mn, b_mn, N, K):
    _run(64, N, K, a_mn, b_mn, d_lane=d_lane)
