"""CPU tests of the C-ABI library: it loads without a GPU, exports every
symbol include/fftconv.h declares, validates arguments before any launch, and
its host planner (Eq. 2 cost model, factorisation, sparsity mask) matches the
paper's printed values."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2311_05908_b200 import _abi, build
    build.build()  # in-tree nvcc build (cross-compiles without a GPU)
    return _abi.lib()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "fftconv.h")).read()
    declared = set(re.findall(r"^(?:fftconv_status_t|void|const char\*|int64_t|int32_t|double)\s+(fftconv_[a-z0-9_]+)\s*\(",
                              hdr, re.M))
    assert {"fftconv_plan", "fftconv_precompute_kf", "fftconv_fwd", "fftconv_gated_fwd", "fftconv_bwd"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    from paper_2311_05908_b200 import _abi
    assert set(_abi.ABI_SYMBOLS) == declared


def _plan(lib, N, L, dtype=0, causal=1, sp=None):
    h = ctypes.c_void_p()
    rc = lib.fftconv_plan(ctypes.byref(h), N, L, dtype, causal, sp)
    return rc, h


def test_plan_validation(lib):
    assert _plan(lib, 1000, 2000)[0] == 2                 # not a power of two
    assert _plan(lib, 1024, 3000)[0] == 2
    assert _plan(lib, 0, 2048)[0] == 1                    # invalid
    assert _plan(lib, 1024, 2048, dtype=9)[0] == 1
    assert _plan(lib, 1024, 2048, causal=0)[0] == 1       # circular needs fft_size == N
    rc, h = _plan(lib, 1024, 2048)
    assert rc == 0
    lib.fftconv_plan_destroy(h)
    rc, h = _plan(lib, 1024, 1024, causal=0)
    assert rc == 0
    lib.fftconv_plan_destroy(h)
    assert lib.fftconv_last_error() is not None


@pytest.mark.parametrize("N,fft,causal", [(1024, 2048, 1), (2048, 4096, 1), (4096, 8192, 1), (8192, 16384, 1),
                                          (1 << 15, 1 << 16, 1),
                                          (1 << 20, 1 << 21, 1), (1 << 22, 1 << 23, 1), (1 << 23, 1 << 23, 0),
                                          (1 << 20, 16384, 1)])
def test_plan_info_factors_cover_L(lib, N, fft, causal):
    """plan_info reports every level: prod(factors[:order]) == fft_size for
    fused, one-level, recursive (up to three outer levels) and partial plans."""
    from paper_2311_05908_b200 import _abi
    rc, h = _plan(lib, N, fft, causal=causal)
    assert rc == 0
    info = _abi.PlanInfo()
    assert lib.fftconv_plan_info(h, ctypes.byref(info)) == 0
    assert 2 <= info.order <= len(info.factors)
    assert int(np.prod([info.factors[i] for i in range(info.order)])) == fft
    lib.fftconv_plan_destroy(h)


def test_plan_info_and_calls_without_upload(lib):
    from paper_2311_05908_b200 import _abi
    rc, h = _plan(lib, 1024, 2048)
    info = _abi.PlanInfo()
    assert lib.fftconv_plan_info(h, ctypes.byref(info)) == 0
    assert (info.N, info.fft_size, info.causal, info.regime, info.order) == (1024, 2048, 1, 1, 2)
    assert info.factors[0] * info.factors[1] == 2048
    assert info.max_kernel_len == 1024
    assert info.table_bytes > 0 and info.kf_bytes_per_head >= 2048 * 8
    # argument errors are caught before any CUDA call (no GPU here)
    assert lib.fftconv_fwd(h, None, None, None, 1, 1, None, None) == 1
    assert lib.fftconv_precompute_kf(h, None, 1, 1, None, None) == 1
    assert lib.fftconv_plan_upload(None, None, None) == 1
    lib.fftconv_plan_destroy(h)


def test_factorize_examples(lib):
    # SPEC S:210-212 examples of the balanced split
    out = (ctypes.c_int64 * 4)()
    for n, p, exp in [(4096, 3, [16, 16, 16]), (1024, 2, [32, 32]), (2 ** 22, 4, [64, 64, 32, 32])]:
        k = lib.fftconv_factorize(n, p, out)
        assert list(out[:k]) == exp


def test_cost_model_reproduces_paper_order_grouping(lib, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "order_selection_a100.json")))
    c = g["constants"]
    args = [c["mu"], c["sigma_H"], c["sigma_S"], c["tau_M"], c["tau_G"], c["sram_bytes"]]
    for n, p in g["expected_p"].items():
        assert lib.fftconv_select_order(int(n), *args) == p, n
    # Eq. 2 compute term example: n=4096, p=2 -> 2*16*4096*64/234e12 s
    cost = lib.fftconv_cost_eq2(4096, 2, *args)
    flop = 2 * 16 * 4096 * 64 / 234e12
    io = 2 * 4 * 4096 / 9.5e12
    assert abs(cost - (flop + io)) < 1e-15
    # linear growth O(N^{(p+1)/p}) of the flop term for equal factors
    c1 = lib.fftconv_cost_eq2(2 ** 12, 2, 1, 1e30, 1e30, 1.0, 1.0, 1e30)
    c2 = lib.fftconv_cost_eq2(2 ** 16, 2, 1, 1e30, 1e30, 1.0, 1.0, 1e30)
    assert abs(c2 / c1 - (2 ** 16 / 2 ** 12) ** 1.5) < 1e-9


def test_sparsity_mask_matches_oracle_reading(lib):
    """The planner's Hermitian-symmetric mask (A13) has the same zero
    fraction as the oracle's independently written mask."""
    from paper_2311_05908_b200 import _abi
    L = 2048
    dims = [32, 64]
    zeroed = [16, 32]
    keeps = orc.keep_masks_from_zero_counts(dims, zeroed)
    sp = _abi.Sparsity()
    sp.ndims = 2
    bufs = []
    for j, (d, kp) in enumerate(zip(dims, keeps)):
        sp.dims[j] = d
        b = (ctypes.c_uint8 * d)(*[int(x) for x in kp])
        bufs.append(b)
        sp.keep[j] = ctypes.cast(b, ctypes.POINTER(ctypes.c_uint8))
    h = ctypes.c_void_p()
    assert lib.fftconv_plan(ctypes.byref(h), 1024, L, 0, 1, ctypes.byref(sp)) == 0
    info = _abi.PlanInfo()
    lib.fftconv_plan_info(h, ctypes.byref(info))
    m = orc.frequency_mask(dims, keeps)
    assert abs(info.mask_fraction - (1.0 - m.mean())) < 1e-12
    lib.fftconv_plan_destroy(h)
    sp.dims[0] = 31
    assert lib.fftconv_plan(ctypes.byref(h), 1024, L, 0, 1, ctypes.byref(sp)) == 4


def _sparse_plan(lib, N, dims, keeps, dtype=0):
    from paper_2311_05908_b200 import _abi
    sp = _abi.Sparsity()
    sp.ndims = len(dims)
    bufs = []
    for j, (d, kp) in enumerate(zip(dims, keeps)):
        sp.dims[j] = d
        b = (ctypes.c_uint8 * d)(*[int(x) for x in kp])
        bufs.append(b)
        sp.keep[j] = ctypes.cast(b, ctypes.POINTER(ctypes.c_uint8))
    h = ctypes.c_void_p()
    assert lib.fftconv_plan(ctypes.byref(h), N, 2 * N, dtype, 1, ctypes.byref(sp)) == 0
    info = _abi.PlanInfo()
    lib.fftconv_plan_info(h, ctypes.byref(info))
    lib.fftconv_plan_destroy(h)
    return info


@pytest.mark.parametrize("N", [1024, 8192, 16384, 32768, 1 << 20])
def test_slow_digit_skip_fraction(lib, N):
    """A symmetric low-pass mask (keep |f| < L/8, A13) zeroes the middle two
    of the four chunks of 8 stage-B columns k1 of the inner transform
    (f = k0 + L0 (k2 + 64 k1)): the planner skips them and
    reports skip_fraction 0.5; the oracle's mask confirms which chunks are
    all-zero.  A dense-chunk mask (trailing zeros of the FAST digit) skips
    no chunk."""
    L = 2 * N
    dims = [16, L // 16]
    keeps = orc.keep_masks_from_zero_counts(dims, [14, 0])
    m = orc.frequency_mask(dims, keeps)
    span = L // 4
    assert [bool(m[c * span:(c + 1) * span].any()) for c in range(4)] == [True, False, False, True]
    info = _sparse_plan(lib, N, dims, keeps)
    assert abs(info.skip_fraction - 0.5) < 1e-12
    assert abs(info.mask_fraction - (1 - m.mean())) < 1e-12
    # fp32 validation plans never skip stage-B chunks
    if N <= 16384:
        assert _sparse_plan(lib, N, dims, keeps, dtype=2).skip_fraction == 0.0
    # a fast-digit mask (keep f mod 16 < 2) leaves every chunk live; one-level
    # multipass plans skip its all-zero outer rows k0 = f mod L0 instead
    dims2 = [L // 16, 16]
    keeps2 = orc.keep_masks_from_zero_counts(dims2, [0, 14])
    m2 = orc.frequency_mask(dims2, keeps2)
    L0 = L // 2048
    rows = 1.0 if L0 == 1 else np.mean([m2[k0::L0].any() for k0 in range(L0)])
    expect = 1.0 - rows if 1 < L0 <= 16 else 0.0
    assert abs(_sparse_plan(lib, N, dims2, keeps2).skip_fraction - expect) < 1e-12


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2311_05908_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_f32_validation_plans(lib):
    # the fp32 validation build: fused and one-level multipass sizes plan;
    # recursive (fft_size > 32768) does not
    for N, L in ((256, 512), (1024, 2048), (8192, 16384)):
        rc, h = _plan(lib, N, L, dtype=2)
        assert rc == 0, (N, L)
        lib.fftconv_plan_destroy(h)
    assert _plan(lib, 32768, 65536, dtype=2)[0] == 5


def test_b200_cost_model_predicts_sweep(lib):
    """NEXT-1: the library's B200 tier cost model (default coefficients,
    fitted by tools/cost_model.py) predicts every measured bench step within
    +-20 % (tests/golden/b200_step_times.json: the sweep of one B200 run,
    k_f precompute + convolution), and the planner uses it to choose the
    single-pass order-3 regime at fft_size 4096 / 8192."""
    import bench
    from paper_2311_05908_b200 import _abi
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "b200_step_times.json")))
    assert len(g["ms_per_step"]) >= 20
    for name, ms in g["ms_per_step"].items():
        wl = bench.WORKLOADS[name]
        dt = {"f16": 0, "bf16": 1}[wl["dtype"]]
        sp = None
        if wl["sparse"]:
            dims, keeps = bench.sparsity_spec(wl["sparse"], wl["fft"])
            sp = _abi.Sparsity()
            sp.ndims = len(dims)
            bufs = []
            for j, (d, kp) in enumerate(zip(dims, keeps)):
                sp.dims[j] = int(d)
                bufs.append((ctypes.c_uint8 * int(d))(*[1 if q else 0 for q in kp]))
                sp.keep[j] = ctypes.cast(bufs[-1], ctypes.POINTER(ctypes.c_uint8))
        h = ctypes.c_void_p()
        assert lib.fftconv_plan(ctypes.byref(h), wl["N"], wl["fft"], dt, int(wl["causal"]),
                                ctypes.byref(sp) if sp is not None else None) == 0
        t = ctypes.c_double()
        assert lib.fftconv_cost_predict(h, wl["B"], wl["H"], int(wl["bwd"]), int(wl["gated"]), None,
                                        ctypes.byref(t)) == 0
        lib.fftconv_plan_destroy(h)
        assert abs(t.value * 1e3 / ms - 1) <= 0.20, (name, t.value * 1e3, ms)
    for N in (2048, 4096):
        rc, h = _plan(lib, N, 2 * N)
        info = _abi.PlanInfo()
        assert lib.fftconv_plan_info(h, ctypes.byref(info)) == 0
        assert info.order == 3 and info.regime == 1
        lib.fftconv_plan_destroy(h)
