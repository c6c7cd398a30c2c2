"""fftconv_fwd_host (end-to-end from host buffers, copies of neighbouring
batch chunks overlapped with the convolution): results are bitwise those of
the device call, for ragged chunking and for the fused and multipass regimes."""
import numpy as np
import pytest

import synth

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
