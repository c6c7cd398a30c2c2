"""fp32 validation build (north star: "<= 1e-5 relative L2 on an fp32
validation build"): the same plan, packing, Monarch decomposition, causal
skipping, k_f layout and multipass outer passes as the fp16/bf16 path, with
every stage in fp32 on the CUDA cores (kernels_f32.cu, fp32 intermediates in
kernels_mp.cu).  Compared element by element with the fp64 oracle on the
same fp32 inputs."""
import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity_f32

torch = pytest.importorskip("torch")

REL_L2 = 1e-5


def _run(N, causal, gated, B, H, seed, fft_size=None, K=None):
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, fft_size=fft_size, dtype=torch.float32, causal=causal)
    K = K or N
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f32")
    u = q("u")
    k = synth.decay_filters(seed, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda")
    kf = plan.precompute_kf(t(k))
    if gated:
        w, v = q("w"), q("v")
        y = plan.gated_fwd(t(u), t(w), t(v), kf)
        ref = orc.conv_fwd(u, k.astype(np.float64), causal=causal, w=w, v=v)
    else:
        y = plan.fwd(t(u), kf)
        ref = orc.conv_fwd(u, k.astype(np.float64), causal=causal)
    torch.cuda.synchronize()
    got = y.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got))
    rel, _ = assert_parity_f32(got, ref)
    return rel, plan


@pytest.mark.gpu
@pytest.mark.parametrize("N", [256, 512, 1024])
@pytest.mark.parametrize("gated", [False, True])
def test_f32_fused_causal(N, gated):
    rel, plan = _run(N, True, gated, B=5, H=3, seed=21)
    assert plan.info.regime == 1
    assert rel <= REL_L2, rel


@pytest.mark.gpu
@pytest.mark.parametrize("N", [512, 2048])
def test_f32_fused_circular(N):
    rel, _ = _run(N, False, True, B=4, H=2, seed=22)
    assert rel <= REL_L2, rel


@pytest.mark.gpu
@pytest.mark.parametrize("N", [2048, 4096, 8192, 16384])
@pytest.mark.parametrize("gated", [False, True])
def test_f32_multipass(N, gated):
    rel, plan = _run(N, True, gated, B=3, H=2, seed=23)
    assert plan.info.regime == 3
    assert rel <= REL_L2, rel


@pytest.mark.gpu
def test_f32_partial():
    rel, plan = _run(16384, True, False, B=2, H=2, seed=24, fft_size=4096, K=1500)
    assert plan.info.regime == 2
    assert rel <= REL_L2, rel


@pytest.mark.gpu
def test_f32_sparse_multipass():
    """fp32 validation build with a frequency-sparse plan (masked k_f rows
    are zero-filled; the fp32 inner pass transforms every row)."""
    from paper_2311_05908_b200 import FFTConvPlan
    N, B, H = 16384, 3, 2
    keep_k0 = np.zeros(16, bool)
    keep_k0[[0, 1, 8, 15]] = True
    dims, keeps = [2048, 16], [np.ones(2048, bool), keep_k0]
    plan = FFTConvPlan(N, dtype=torch.float32, causal=True, sparsity=(dims, keeps))
    u = synth.quantize(synth.signal(25, "u", B, H, N), "f32")
    k = synth.decay_filters(25, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(torch.tensor(u, dtype=torch.float32, device="cuda"), kf).cpu().numpy()
    ref = orc.conv_fwd(u, k.astype(np.float64), mask=orc.frequency_mask(dims, keeps))
    rel, _ = assert_parity_f32(y, ref)
    assert rel <= REL_L2, rel


@pytest.mark.gpu
@pytest.mark.parametrize("N,causal,fft,K,gated", [(1024, True, None, None, True), (512, False, None, None, False),
                                                  (8192, True, None, None, True), (16384, True, 4096, 1500, False)])
def test_f32_backward(N, causal, fft, K, gated):
    """fp32 validation build of the backward (same passes, CUDA-core fp32
    inner): du, dw, dv and dk against the fp64 oracle at 1e-5."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, seed = 3, 2, 41
    plan = FFTConvPlan(N, fft_size=fft, dtype=torch.float32, causal=causal)
    K = K or N
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f32")
    u, dy = q("u"), q("dy")
    w, v = (q("w"), q("v")) if gated else (None, None)
    k = synth.decay_filters(seed, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda") if a is not None else None
    kf = plan.precompute_kf(t(k))
    g = plan.bwd(t(dy), t(u), kf, K, w=t(w), v=t(v))
    torch.cuda.synchronize()
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), causal=causal, w=w, v=v)
    for key in ("du", "dw", "dv", "dk"):
        if ref[key] is None:
            continue
        got = g[key].cpu().numpy().astype(np.float64)
        rel, _ = assert_parity_f32(got, ref[key], key)
        assert rel <= REL_L2, (key, rel)
