"""fftconv_fwd_host (end-to-end from host buffers, copies of neighbouring
batch chunks overlapped with the convolution): results are bitwise those of
the device call, for ragged chunking and for the fused and multipass regimes."""
import numpy as np
import pytest

import synth
from parity import assert_parity

torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("N,gated,B,rpc", [(1024, True, 7, 2), (1024, False, 5, 8), (8192, True, 5, 2),
                                           (8192, False, 3, 1)])
def test_fwd_host_matches_device(N, gated, B, rpc):
    from paper_2311_05908_b200 import FFTConvPlan
    H, dt = 3, torch.float16
    plan = FFTConvPlan(N, dtype=dt, causal=True)
    q = lambda name: torch.tensor(synth.quantize(synth.signal(5, name, B, H, N), "f16"), dtype=dt)
    u, w, v = q("u"), q("w"), q("v")
    k = torch.tensor(synth.decay_filters(5, H, N).astype(np.float32), device="cuda")
    kf = plan.precompute_kf(k)
    if gated:
        ref = plan.gated_fwd(u.cuda(), w.cuda(), v.cuda(), kf)
        got = plan.fwd_host(u.pin_memory(), kf, w=w.pin_memory(), v=v.pin_memory(), rows_per_chunk=rpc)
    else:
        ref = plan.fwd(u.cuda(), kf)
        got = plan.fwd_host(u.pin_memory(), kf, rows_per_chunk=rpc)
    torch.cuda.synchronize()
    assert torch.equal(got, ref.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_fwd_stream_partial_long_rows(dtype, gated):
    """fftconv_fwd_stream (NEXT-4): rows of N_total = 32768 streamed through a
    partial plan with N = 8192, fft_size 4096 (C = 2048, segments of 6144
    outputs, the last one ragged) equal the causal convolution of the whole
    rows with the truncated filter (K = 700)."""
    from oracle import oracle as orc
    from paper_2311_05908_b200 import FFTConvPlan
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16}[dtype]
    B, H, NT, K = 2, 3, 32768, 700
    plan = FFTConvPlan(8192, fft_size=4096, dtype=tdt, causal=True)
    assert plan.info.regime == 2
    q = lambda name: synth.quantize(synth.signal(15, name, B, H, NT), dtype)
    u, w, v = q("u"), q("w"), q("v")
    k = synth.decay_filters(15, H, K).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    th = lambda a: torch.tensor(a, dtype=tdt).pin_memory()
    if gated:
        y = plan.fwd_stream(th(u), kf, w=th(w), v=th(v))
        ref = orc.conv_fwd(u, k.astype(np.float64), w=w, v=v)
    else:
        y = plan.fwd_stream(th(u), kf)
        ref = orc.conv_fwd(u, k.astype(np.float64))
    torch.cuda.synchronize()
    got = y.float().numpy().astype(np.float64)
    assert_parity(got, ref)
