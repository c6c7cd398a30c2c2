"""GPU parity of the bidirectional (two-sided) convolution, reading B1
(SURVEY 8(f) NEXT-4): k_f of the two-sided filter from
fftconv_precompute_kf_bidir through the unchanged forward regimes (fused
order 2, single-pass order 3, one-level multipass, recursive multipass) and
fftconv_bwd_bidir, against the fp64 oracle (conv_fwd_bidir /
conv_bwd_bidir), element by element."""
import ctypes

import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity, assert_parity_f32

torch = pytest.importorskip("torch")

TDT = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}


def _inputs(N, K, B, H, dtype, gated, seed):
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), dtype)
    u, dy = q("u"), q("dy")
    w = q("w") if gated else None
    v = q("v") if gated else None
    kf = synth.decay_filters(seed, H, K).astype(np.float32)
    kb = synth.decay_filters(seed + 7, H, K).astype(np.float32)
    return u, w, v, dy, kf, kb


def _dev(a, dtype):
    return torch.tensor(a, dtype=TDT[dtype], device="cuda") if a is not None else None


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(256, 256), (1024, 1024), (1024, 100), (2048, 2048), (4096, 333),
                                 (8192, 8192), (32768, 32768)])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_bidir_fwd(N, K, dtype, gated):
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 3, 2
    u, w, v, _, kf, kb = _inputs(N, K, B, H, dtype, gated, seed=N + K)
    plan = FFTConvPlan(N, dtype=TDT[dtype], causal=True)
    kfd = plan.precompute_kf_bidir(torch.tensor(kf, device="cuda"), torch.tensor(kb, device="cuda"))
    if gated:
        y = plan.gated_fwd(_dev(u, dtype), _dev(w, dtype), _dev(v, dtype), kfd)
    else:
        y = plan.fwd(_dev(u, dtype), kfd)
    torch.cuda.synchronize()
    ref = orc.conv_fwd_bidir(u, kf.astype(np.float64), kb.astype(np.float64), w=w, v=v)
    assert_parity(y.float().cpu().numpy(), ref, f"bidir fwd N={N} K={K}")


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(1024, 1024), (2048, 700), (8192, 8192), (32768, 32768)])
@pytest.mark.parametrize("gated", [False, True])
def test_bidir_bwd(N, K, gated):
    from paper_2311_05908_b200 import FFTConvPlan
    dtype = "f16"
    B, H = 3, 2
    u, w, v, dy, kf, kb = _inputs(N, K, B, H, dtype, gated, seed=3 * N + K)
    plan = FFTConvPlan(N, dtype=TDT[dtype], causal=True)
    kfd = plan.precompute_kf_bidir(torch.tensor(kf, device="cuda"), torch.tensor(kb, device="cuda"))
    g = plan.bwd_bidir(_dev(dy, dtype), _dev(u, dtype), kfd, K, w=_dev(w, dtype), v=_dev(v, dtype))
    torch.cuda.synchronize()
    ref = orc.conv_bwd_bidir(dy, u, kf.astype(np.float64), kb.astype(np.float64), w=w, v=v)
    for key in ("du", "dw", "dv", "dk_fwd", "dk_bwd"):
        if ref[key] is None:
            assert g[key] is None
            continue
        assert_parity(g[key].float().cpu().numpy(), ref[key], f"bidir bwd {key} N={N}")


@pytest.mark.gpu
def test_bidir_f32_validation_build():
    from paper_2311_05908_b200 import FFTConvPlan
    N, K, B, H = 1024, 1024, 2, 3
    u, w, v, dy, kf, kb = _inputs(N, K, B, H, "f32", True, seed=11)
    plan = FFTConvPlan(N, dtype=torch.float32, causal=True)
    kfd = plan.precompute_kf_bidir(torch.tensor(kf, device="cuda"), torch.tensor(kb, device="cuda"))
    y = plan.gated_fwd(_dev(u, "f32"), _dev(w, "f32"), _dev(v, "f32"), kfd)
    g = plan.bwd_bidir(_dev(dy, "f32"), _dev(u, "f32"), kfd, K, w=_dev(w, "f32"), v=_dev(v, "f32"))
    torch.cuda.synchronize()
    k64, b64 = kf.astype(np.float64), kb.astype(np.float64)
    assert_parity_f32(y.cpu().numpy(), orc.conv_fwd_bidir(u, k64, b64, w=w, v=v), "bidir f32 fwd")
    ref = orc.conv_bwd_bidir(dy, u, k64, b64, w=w, v=v)
    for key in ("du", "dw", "dv", "dk_fwd", "dk_bwd"):
        assert_parity_f32(g[key].cpu().numpy(), ref[key], f"bidir f32 {key}")


@pytest.mark.gpu
def test_bidir_reduces_to_causal():
    # k_bwd = 0: bitwise the causal k_f's forward
    from paper_2311_05908_b200 import FFTConvPlan
    N, K, B, H = 2048, 2048, 4, 2
    u, _, _, _, kf, _ = _inputs(N, K, B, H, "f16", False, seed=5)
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True)
    kt = torch.tensor(kf, device="cuda")
    y1 = plan.fwd(_dev(u, "f16"), plan.precompute_kf_bidir(kt, torch.zeros_like(kt)))
    y0 = plan.fwd(_dev(u, "f16"), plan.precompute_kf(kt))
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


@pytest.mark.gpu
@pytest.mark.parametrize("N,fft,causal", [(8192, 4096, True), (1024, 1024, False)])
def test_bidir_rejects_partial_and_circular(N, fft, causal):
    from paper_2311_05908_b200 import FFTConvPlan, _abi
    plan = FFTConvPlan(N, fft_size=fft, dtype=torch.float16, causal=causal)
    k = torch.zeros(2, 16, device="cuda")
    with pytest.raises(_abi.FFTConvError) as e:
        plan.precompute_kf_bidir(k, k)
    assert e.value.status == 5  # FFTCONV_ERR_UNSUPPORTED
