"""NEXT-1: the paper's cost-model constants re-measured on B200 and the B200
tier cost model fitted to the bench sweep.

  python tools/cost_model.py measure OUT.json        (GPU) sigma_H, sigma_S, tau_M, tau_G
  python tools/cost_model.py fit BENCH.json [CONST.json] [--md OUT.md]
                                                     (CPU) fit + predicted-vs-measured table

Protocol of P:786-791 (tab:gpu_costs): sigma_H = torch.clone of a large
tensor; tau_M = a real fp16 matrix multiply; tau_G = continuously applying
twiddle factors (selftest kernel twiddle_rate_kernel, f32x2 complex
multiplies); sigma_S = shared-memory write/read bandwidth between compute
steps (selftest kernel smem_bw_kernel).

The fit uses the library's own work-unit counts (fftconv_cost_features,
host only) for each bench workload and non-negative least squares on the
relative error of the step time (k_f precompute + convolution).  Points are
split into a fit set and a held-out set; the table reports both.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NFEAT = 12
FEAT_NAMES = ["o2 causal tiles", "o2 circular tiles", "o3 L0=2 tiles", "o3 L0=4 tiles", "outer-pass elems",
              "k_f elems", "launches", "bwd tiles", "bwd T-chain elems", "dk elems", "gated tiles", "HBM bytes"]
HELD_OUT = {"gsweep4096", "gsweep8192", "cfg5", "circ16384", "sweep32768", "sweep262144", "cfg4"}


def measure(out_path):
    import torch
    dev = torch.device("cuda")
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2311_05908_b200", "libfftconv_selftest.so"))
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            a, b = ev(), ev()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        return best

    x = torch.empty(1 << 30, dtype=torch.float16, device=dev)
    t = timed(lambda: x.clone())
    sigma_h = 2 * x.numel() * 2 / t
    del x
    a = torch.randn(8192, 8192, dtype=torch.float16, device=dev)
    t = timed(lambda: torch.matmul(a, a))
    tau_m = 2 * 8192 ** 3 / t
    del a
    sink = torch.zeros(256, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 4096
    t = timed(lambda: lib.fcst_twiddle_rate(blocks, iters, ctypes.c_void_p(sink.data_ptr()), stream))
    tau_g = blocks * 256 * iters * (16 + 2) * 6 / t  # 16 data + 2 twiddle complex products, 6 flops each
    t = timed(lambda: lib.fcst_smem_bw(blocks, iters, ctypes.c_void_p(sink.data_ptr()), stream))
    sigma_s = blocks * 256 * iters * 8 * 32 / t  # 8 steps x (16 B store + 16 B load)
    out = {"sigma_H": sigma_h, "sigma_S": sigma_s, "tau_M": tau_m, "tau_G": tau_g, "sms": sms,
           "how": "P:786-791 protocol on B200: torch.clone 2 GiB, fp16 matmul 8192^3, selftest twiddle_rate "
                  "and smem_bw kernels (best of 10, CUDA events)"}
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps(out, indent=1))


def _features(lib, wl):
    from paper_2311_05908_b200 import _abi
    dt = {"f16": _abi.FFTCONV_F16, "bf16": _abi.FFTCONV_BF16}[wl["dtype"]]
    h = ctypes.c_void_p()
    sp = None
    if wl.get("sparse"):
        import bench
        dims, keeps = bench.sparsity_spec(wl["sparse"], wl["fft"])
        sp = _abi.Sparsity()
        sp.ndims = len(dims)
        bufs = []
        for j, (d, kp) in enumerate(zip(dims, keeps)):
            sp.dims[j] = int(d)
            b = (ctypes.c_uint8 * int(d))(*[1 if q else 0 for q in kp])
            bufs.append(b)
            sp.keep[j] = ctypes.cast(b, ctypes.POINTER(ctypes.c_uint8))
    _abi.check(lib.fftconv_plan(ctypes.byref(h), wl["N"], wl["fft"], dt, int(wl["causal"]),
                                ctypes.byref(sp) if sp is not None else None))
    f = (ctypes.c_double * NFEAT)()
    _abi.check(lib.fftconv_cost_features(h, wl["B"], wl["H"], int(wl["bwd"]), int(wl["gated"]), f))
    lib.fftconv_plan_destroy(h)
    return np.array(f[:])


def eq2_seconds(wl, c):
    """Eq. 2 with B200 constants: C = BH sum_i [16 N N_i / gamma + 4N / omega]
    for the best balanced order p <= 4 of N = fft_size (A10/A11; mu = 16,
    SRAM working set 227 KB per SM)."""
    from paper_2311_05908_b200 import _abi
    lib = _abi.lib()
    L = wl["fft"]
    best = min(x for x in (lib.fftconv_cost_eq2(L, p, 16.0, c["sigma_H"], c["sigma_S"], c["tau_M"], c["tau_G"],
                                                 227.0 * 1024) for p in (2, 3, 4)) if x > 0)
    rows = wl["B"] * wl["H"] * (wl["N"] // (L // 2) if wl["causal"] and L < 2 * wl["N"] else 1)
    return best * rows * (3.0 if wl["bwd"] else 1.0)


def fit(bench_paths, const_path=None, md_path=None):
    import bench
    from paper_2311_05908_b200 import _abi
    lib = _abi.lib()
    meas = {}
    for bp in bench_paths:
        for line in open(bp):
            line = line.strip()
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            if "sweep" in d:
                for name, v in d["sweep"].items():
                    if "ms_per_step" in v:
                        meas[name] = v["ms_per_step"] * 1e-3
    names = sorted(meas)
    X = np.array([_features(lib, bench.WORKLOADS[n]) for n in names])
    y = np.array([meas[n] for n in names])
    fit_idx = [i for i, n in enumerate(names) if n not in HELD_OUT]
    from scipy.optimize import nnls
    A = X[fit_idx] / y[fit_idx, None]
    coef, _ = nnls(A, np.ones(len(fit_idx)))
    pred = X @ coef
    const = json.load(open(const_path)) if const_path and os.path.exists(const_path) else None
    lines = ["| workload | set | measured ms | B200 model ms | error | paper Eq. 2 (B200 constants) ms |",
             "|---|---|---|---|---|---|"]
    worst = 0.0
    for i, n in enumerate(names):
        err = pred[i] / y[i] - 1
        worst = max(worst, abs(err))
        e2 = eq2_seconds(bench.WORKLOADS[n], const) * 1e3 if const else float("nan")
        lines.append(f"| {n} | {'held out' if n in HELD_OUT else 'fit'} | {y[i] * 1e3:.4f} | {pred[i] * 1e3:.4f} | "
                     f"{100 * err:+.1f} % | {e2:.4f} |")
    lines.append("")
    lines.append("coefficients (s per unit): " + ", ".join(f"{FEAT_NAMES[k]} {coef[k]:.4g}" for k in range(NFEAT)))
    lines.append(f"worst |error| {100 * worst:.1f} %")
    txt = "\n".join(lines)
    print(txt)
    print("\n// plan.cpp defaults")
    for k in range(NFEAT):
        print(f"#define COST_B200_{k} {coef[k]:.6e}")
    if md_path:
        with open(md_path, "w") as fh:
            fh.write("# B200 cost model: predicted vs measured (step = k_f precompute + conv)\n\n")
            if const:
                fh.write("Measured constants (P:786-791 protocol): " + ", ".join(
                    f"{k} {const[k]:.4g}" for k in ("sigma_H", "sigma_S", "tau_M", "tau_G")) + "\n\n")
            fh.write(txt + "\n")
    return coef


if __name__ == "__main__":
    if sys.argv[1] == "measure":
        measure(sys.argv[2])
    else:
        args = sys.argv[2:]
        md = None
        if "--md" in args:
            md = args[args.index("--md") + 1]
            args = args[:args.index("--md")]
        const = [a for a in args if "const" in a]
        benches = [a for a in args if a not in const]
        fit(benches, const[0] if const else None, md)
