"""GPU parity of the fused forward kernels against the fp64 oracle.

Inputs are seeded synthetic (synth/), quantised to the I/O dtype on the host
so both sides consume identical values.  Bar (BASELINE.json north_star):
rel-L2 <= 2e-3 and max-abs <= 1e-2 * max|y| for fp16/bf16 I/O."""
import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity, assert_parity_f32  # noqa: F401

torch = pytest.importorskip("torch")

REL_L2 = 2e-3
MAX_ABS = 1e-2

TDT = {"f16": torch.float16, "bf16": torch.bfloat16}


def _run(N, causal, dtype, gated, B, H, seed=0, filt="decay"):
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, dtype=TDT[dtype], causal=causal)
    K = N
    u = synth.quantize(synth.signal(seed, "u", B, H, N), dtype)
    k = (synth.decay_filters(seed, H, K) if filt == "decay" else synth.flat_filters(seed, H, K)).astype(np.float32)
    dev = "cuda"
    tu = torch.tensor(u, dtype=TDT[dtype], device=dev)
    tk = torch.tensor(k, device=dev)
    kf = plan.precompute_kf(tk)
    if gated:
        w = synth.quantize(synth.signal(seed, "w", B, H, N), dtype)
        v = synth.quantize(synth.signal(seed, "v", B, H, N), dtype)
        y = plan.gated_fwd(tu, torch.tensor(w, dtype=TDT[dtype], device=dev),
                           torch.tensor(v, dtype=TDT[dtype], device=dev), kf)
        ref = orc.conv_fwd(u, k.astype(np.float64), causal=causal, w=w, v=v)
    else:
        y = plan.fwd(tu, kf)
        ref = orc.conv_fwd(u, k.astype(np.float64), causal=causal)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy().astype(np.float64)
    return got, ref


def _assert_close(got, ref):
    return assert_parity(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N", [256, 512, 1024])
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("gated", [False, True])
def test_fwd_causal_parity(N, dtype, gated):
    # B = 37 is ragged (not a multiple of the tile's row count) and odd
    got, ref = _run(N, True, dtype, gated, B=37, H=3)
    _assert_close(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N", [512, 1024, 2048])
@pytest.mark.parametrize("gated", [False, True])
def test_fwd_circular_parity(N, gated):
    got, ref = _run(N, False, "f16", gated, B=6, H=2)
    _assert_close(got, ref)


@pytest.mark.gpu
def test_fwd_cfg1_direct_sum():
    """cfg 1: causal fp16, B=1, H=4, N=256, checked against the direct sum."""
    got, _ = _run(256, True, "f16", False, B=1, H=4, seed=1)
    u = synth.quantize(synth.signal(1, "u", 1, 4, 256), "f16")
    k = synth.decay_filters(1, 4, 256).astype(np.float32).astype(np.float64)
    ref = np.stack([[orc.direct_conv(u[0, h], k[h], True) for h in range(4)]])
    _assert_close(got, ref)


@pytest.mark.gpu
def test_fwd_flat_filter_and_empty():
    got, ref = _run(1024, True, "f16", True, B=2, H=5, filt="flat")
    _assert_close(got, ref)
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(1024)
    kf = plan.precompute_kf(torch.zeros(3, 1024, device="cuda"))
    y = plan.fwd(torch.zeros(0, 3, 1024, dtype=torch.float16, device="cuda"), kf)
    assert y.shape == (0, 3, 1024)


@pytest.mark.gpu
def test_fwd_delta_filter_identity():
    from paper_2311_05908_b200 import FFTConvPlan
    N = 1024
    plan = FFTConvPlan(N)
    k = torch.zeros(2, N, device="cuda")
    k[:, 0] = 1.0
    kf = plan.precompute_kf(k)
    u = torch.tensor(synth.quantize(synth.signal(3, "u", 4, 2, N), "f16"), dtype=torch.float16, device="cuda")
    y = plan.fwd(u, kf)
    err = (y.float() - u.float()).abs().max().item()
    assert err < 2e-3 * u.float().abs().max().item()


@pytest.mark.gpu
def test_fwd_cfg2_full_size_sampled():
    """cfg 2 at full size (gated, B=64, H=768, N=1024, fp16), launch config of
    bench.py; sampled outputs checked one by one against the direct sum."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N = 64, 768, 1024
    plan = FFTConvPlan(N, dtype=torch.float16)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(B * H, 48, replace=False))
    u = synth.quantize(synth.signal(5, "u", B, H, N), "f16")
    w = synth.quantize(synth.signal(5, "w", B, H, N), "f16")
    v = synth.quantize(synth.signal(5, "v", B, H, N), "f16")
    k = synth.decay_filters(5, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.gated_fwd(*(torch.tensor(a, dtype=torch.float16, device="cuda") for a in (u, w, v)), kf)
    y = y.float().cpu().numpy().reshape(B * H, N)
    u2, w2, v2 = u.reshape(B * H, N), w.reshape(B * H, N), v.reshape(B * H, N)
    got, ref = [], []
    for r in rows:
        h = r % H
        for i in rng.choice(N, 8, replace=False):
            ref.append(v2[r, i] * orc.direct_point(u2[r], k[h].astype(np.float64), i, wrow=w2[r]))
            got.append(y[r, i])
    got, ref = np.array(got), np.array(ref)
    assert_parity(got, ref)


# ---------------------------------------------------------------- multipass regime (N >= 2048)
@pytest.mark.gpu
@pytest.mark.parametrize("N", [2048, 4096, 8192, 16384])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("f16", True), ("bf16", True)])
def test_fwd_multipass_parity(N, dtype, gated):
    # odd B exercises the zero-filled partner row of the last pair
    got, ref = _run(N, True, dtype, gated, B=3, H=2)
    _assert_close(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N", [4096, 8192])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_fwd_multipass_forced(N, dtype, gated, monkeypatch):
    """The multipass path at sizes the planner now gives to single-pass
    order 3 (FFTCONV_DIT=0 keeps the three-kernel plan)."""
    monkeypatch.setenv("FFTCONV_DIT", "0")
    from paper_2311_05908_b200 import FFTConvPlan
    assert FFTConvPlan(N, dtype=TDT[dtype]).info.regime == 3
    got, ref = _run(N, True, dtype, gated, B=5, H=2)
    _assert_close(got, ref)


@pytest.mark.gpu
def test_fwd_multipass_cfg3_shape_sampled():
    """cfg 3 shape (gated causal bf16, B=16, H=768, N=8192), sampled outputs
    against the direct sum."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N = 16, 768, 8192
    plan = FFTConvPlan(N, dtype=torch.bfloat16)
    assert plan.info.order == 3  # single-pass order 3 (coupled warpgroups, L0 = 8)
    rng = np.random.default_rng(3)
    u = synth.quantize(synth.signal(7, "u", B, H, N), "bf16")
    w = synth.quantize(synth.signal(7, "w", B, H, N), "bf16")
    v = synth.quantize(synth.signal(7, "v", B, H, N), "bf16")
    k = synth.decay_filters(7, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.gated_fwd(*(torch.tensor(a, dtype=torch.bfloat16, device="cuda") for a in (u, w, v)), kf)
    y = y.float().cpu().numpy().reshape(B * H, N)
    u2, w2, v2 = u.reshape(B * H, N), w.reshape(B * H, N), v.reshape(B * H, N)
    got, ref = [], []
    for r in rng.choice(B * H, 24, replace=False):
        for i in rng.choice(N, 6, replace=False):
            ref.append(v2[r, i] * orc.direct_point(u2[r], k[r % H].astype(np.float64), i, wrow=w2[r]))
            got.append(y[r, i])
    got, ref = np.array(got), np.array(ref)
    assert_parity(got, ref)


# ---------------------------------------------------------------- single-pass order 3 (N = 2048, 4096, 8192)
@pytest.mark.gpu
@pytest.mark.parametrize("N", [2048, 4096, 8192])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("f16", True), ("bf16", False), ("bf16", True)])
def test_fwd_order3_single_pass(N, dtype, gated):
    """fft_size 4096 / 8192 / 16384 in ONE fused launch (plan order 3: the
    DFT over the L0 = fft_size / 2048 decimated inner rows z[n0 + L0 n'] runs
    in the pointwise step; L0 = 8: both warpgroups of a CTA share each row
    pair); B = 37 leaves a ragged last tile (4 or 2 rows per tile, L0 = 8:
    the last pair's partner row zero)."""
    from paper_2311_05908_b200 import FFTConvPlan, launch_count_reset
    plan = FFTConvPlan(N, dtype=TDT[dtype])
    assert plan.info.order == 3 and plan.info.regime == 1
    assert plan.info.factors == (N // 1024, 32, 64)
    launch_count_reset()
    got, ref = _run(N, True, dtype, gated, B=37, H=3, seed=31)
    assert launch_count_reset() == 2  # precompute_kf + one convolution
    _assert_close(got, ref)


# ---------------------------------------------------------------- recursive multipass (N >= 32768)
@pytest.mark.gpu
@pytest.mark.parametrize("N", [32768, 262144])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_fwd_multilevel_parity(N, dtype, gated):
    got, ref = _run(N, True, dtype, gated, B=2, H=1)
    _assert_close(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1 << 20, 1 << 22])
def test_fwd_multilevel_whole_rows(N):
    """N = 1M and 4M (the deepest plans): two whole rows (one packed pair)
    against the oracle's fp64 FFT convolution, every output element."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 2, 1
    plan = FFTConvPlan(N, dtype=torch.float16)
    u = synth.quantize(synth.signal(9, "u", B, H, N), "f16")
    k = synth.decay_filters(9, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(torch.tensor(u, dtype=torch.float16, device="cuda"), kf).float().cpu().numpy()
    ref = orc.conv_fwd(u, k.astype(np.float64))
    assert_parity(y, ref)


def _range_stress_inputs(N, K, amp, seed=19):
    """SURVEY 8(d) range-stress row: u = const amp in every row (the packed
    pair z = amp (1 + i) is as coherent as an input can be, so the DC bin
    of every stage carries amp * sqrt(2) * N / sqrt(L) in the unitary
    scaling), k = delta + small noise."""
    u = np.full((2, 1, N), amp, dtype=np.float64)
    k = np.zeros((1, K))
    k[0, 0] = 1.0
    k[0, 1:] = 1e-2 * synth.normal(seed, 9, np.arange(1), K - 1)[0] / np.sqrt(K)
    return synth.quantize(u, "f16"), k.astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("N,amp", [(8192, 8.0), (1 << 20, 8.0), (1 << 22, 8.0), (1 << 20, 64.0), (1 << 22, 64.0),
                                   (4096, 256.0)])
def test_fwd_range_stress(N, amp):
    """u = const amp, k = delta + noise at N = 8K, 1M and 4M (fp16 I/O, fp16
    tensor-core operands and fp16 multipass intermediate): whole rows.  At
    amp = 64 the unscaled DC bin, amp * sqrt(fft_size / 2) >= 65536, would
    overflow fp16 at N >= 1M; the plan's power-of-two headroom pre-scale
    keeps every intermediate finite up to the documented max|g| = 256."""
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, dtype=torch.float16)
    u, k = _range_stress_inputs(N, N, amp)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(torch.tensor(u, dtype=torch.float16, device="cuda"), kf).float().cpu().numpy()
    assert_parity(y, orc.conv_fwd(u, k.astype(np.float64)))


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(1024, 300), (512, 17), (2048, 999), (4096, 33), (8192, 1000), (32768, 4097)])
def test_fwd_full_causal_short_filter(N, K):
    """Full causal plans (fft_size = 2N) with a filter shorter than the
    input (Hyena-style K < N): k is zero-padded to fft_size in k_f, the
    result is the causal conv with k[K:] = 0."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 5, 2
    plan = FFTConvPlan(N, fft_size=2 * N, dtype=torch.float16)
    assert plan.info.regime != 2
    q = lambda name: synth.quantize(synth.signal(23, name, B, H, N), "f16")
    u, w, v = q("u"), q("w"), q("v")
    k = synth.decay_filters(23, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.gated_fwd(t(u), t(w), t(v), kf).float().cpu().numpy()
    assert_parity(y, orc.conv_fwd(u, k.astype(np.float64), w=w, v=v))
    ref_direct = np.array([[v[b, h] * orc.direct_conv(u[b, h] * w[b, h], k[h].astype(np.float64), True)
                            for h in range(H)] for b in range(B)])
    assert_parity(y, ref_direct)


# ---------------------------------------------------------------- circular multipass (fft_size == N >= 4096)
@pytest.mark.gpu
@pytest.mark.parametrize("N", [4096, 16384, 65536])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_fwd_circular_multipass_parity(N, dtype, gated):
    """The paper's circular benchmark rows (FFT size = input length,
    P:1243-1244) beyond the fused sizes: outer passes keep every n0."""
    got, ref = _run(N, False, dtype, gated, B=3, H=2)
    _assert_close(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N,fft", [(4096, None), (65536, None), (16384, 4096)])
def test_edge_single_row_and_empty(N, fft):
    """Multipass / recursive / partial plans with B = 1 (the row pairs with a
    zero partner) and H = 1, and empty batches for forward, backward and the
    host entry points (no launch, no error)."""
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, fft_size=fft, dtype=torch.float16)
    K = (fft // 2) if fft else N
    u = synth.quantize(synth.signal(17, "u", 1, 1, N), "f16")
    dy = synth.quantize(synth.signal(17, "dy", 1, 1, N), "f16")
    k = synth.decay_filters(17, 1, K).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    y = plan.fwd(t(u), kf).float().cpu().numpy()
    _assert_close(y.astype(np.float64), orc.conv_fwd(u, k.astype(np.float64)))
    g = plan.bwd(t(dy), t(u), kf, K)
    ref = orc.conv_bwd(dy, u, k.astype(np.float64))
    for key in ("du", "dk"):
        got = g[key].float().cpu().numpy().astype(np.float64)
        assert_parity(got, ref[key], str(key))
    empty = torch.zeros(0, 1, N, dtype=torch.float16, device="cuda")
    assert plan.fwd(empty, kf).shape == (0, 1, N)
    ge = plan.bwd(empty, empty, kf, K)
    assert ge["du"].shape == (0, 1, N) and float(ge["dk"].abs().max()) == 0.0
    assert plan.fwd_host(torch.zeros(0, 1, N, dtype=torch.float16), kf).shape == (0, 1, N)
