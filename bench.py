#!/usr/bin/env python
"""Benchmark of the B200 FlashFFTConv hot path (bench contract).

One step = one pass of the whole hot path over one batch of synthetic input:
fftconv_precompute_kf (k -> k_f; filters change every
training step) + the convolution call(s) of the workload (a3-a11).

Default workload (BASELINE.json configs[1], the metric's configuration at
N=1): cfg2 "M2-BERT-base gated conv B=64 H=768 N=1024 fp16", causal
(fft_size 2048).  Other configs: --workload cfg1|cfg3|cfg4|cfg5|cfg5dense|
sweep<N>.  Multi-GPU (torchrun): every rank processes its own B x H rows of
the workload (weak scaling; rows are independent, no collective on the data
path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fftconv|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _wl(name, B, H, N, gated=False, dtype="f16", bwd=False, fft=None, K=None, sparse=None, causal=True):
    return dict(name=name, B=B, H=H, N=N, gated=gated, causal=causal, dtype=dtype, bwd=bwd,
                fft=fft or (2 * N if causal else N), K=K or N, sparse=sparse)


WORKLOADS = {
    "cfg1": _wl("cfg1: causal fp16 conv B=1 H=4 N=256 (fft_size 512)", 1, 4, 256),
    "cfg2": _wl("cfg2: M2-BERT-base gated causal conv B=64 H=768 N=1024 fp16 (fft_size 2048)", 64, 768, 1024,
                gated=True),
    "cfg3": _wl("cfg3: Hyena-GPT-s gated causal conv B=16 H=768 N=8192 bf16, fwd+bwd", 16, 768, 8192, gated=True,
                dtype="bf16", bwd=True),
    "cfg4": _wl("cfg4: HyenaDNA partial conv B=1 H=256 N=1048576 K=8192 fp16 (fft_size 16384, overlap-save)",
                1, 256, 1 << 20, fft=16384, K=8192),
    "cfg4bwd": _wl("cfg4 fwd+bwd: HyenaDNA partial conv B=1 H=256 N=1048576 K=8192 fp16 (fft_size 16384)",
                   1, 256, 1 << 20, fft=16384, K=8192, bwd=True),
    "long1m": _wl("long gated causal conv B=8 H=96 N=1048576 bf16, fwd+bwd (two outer levels)", 8, 96, 1 << 20,
                  gated=True, dtype="bf16", bwd=True),
    "cfg5": _wl("cfg5: frequency-sparse causal conv B=8 H=768 N=16384 fp16, 75% of inner Monarch rows skipped",
                8, 768, 16384, sparse="rows75"),
    "cfg5dense": _wl("cfg5 dense reference: causal conv B=8 H=768 N=16384 fp16", 8, 768, 16384),
    "cfg5a": _wl("cfg5a: frequency-sparse causal conv B=8 H=768 N=16384 fp16, symmetric low-pass |f| < L/8 "
                 "(mask 75%), 2 of 4 stage-B column chunks skipped", 8, 768, 16384, sparse="lowpass8"),
    "sp1m91": _wl("frequency-sparse causal conv B=8 H=96 N=1048576 fp16, tab:sparsity_fraction a=b=c=d=16 "
                  "on the 32x32x32x64 grid (P:1035, P:1053-1058)", 8, 96, 1 << 20, sparse="paper:16,16,16,16"),
    "sp1m_lp": _wl("frequency-sparse causal conv B=8 H=96 N=1048576 fp16, symmetric low-pass |f| < L/8",
                   8, 96, 1 << 20, sparse="lowpass8"),
    "cfg5b": _wl("cfg5b: causal conv B=8 H=96 N=4194304 fp16 (fft_size 8M, three outer levels)", 8, 96, 1 << 22),
}
for _n in (256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536):
    WORKLOADS[f"sweep{_n}"] = _wl(f"sweep: causal fp16 conv B*H=49152 N={_n}", 64, 768, _n)
# constant elements (B*H = 49152 * 65536 / N) with B >= 8 (k_f is
# fp32 per head, so B=1 rows would be dominated by k_f bytes)
for _n, _b, _h in ((1 << 18, 16, 768), (1 << 20, 8, 384), (1 << 22, 8, 96)):
    WORKLOADS[f"sweep{_n}"] = _wl(f"sweep: causal fp16 conv B={_b} H={_h} N={_n}", _b, _h, _n)
# gated fp16 sweep points (B=64, H=768): cfg2's path at other N
for _n in (256, 512, 2048, 4096, 8192, 16384):
    WORKLOADS[f"gsweep{_n}"] = _wl(f"sweep: gated causal fp16 conv B*H=49152 N={_n}", 64, 768, _n, gated=True)
# default sweep carried in the bench line (every regime of the metric)
SWEEP = ["sweep256", "sweep512", "sweep1024", "sweep2048", "sweep4096", "sweep8192", "sweep16384",
         "sweep32768", "sweep65536", "sweep262144", "sweep1048576", "sweep4194304",
         "gsweep512", "gsweep2048", "gsweep4096", "gsweep8192", "cfg3", "cfg4", "cfg4bwd", "cfg5", "cfg5a", "cfg5dense", "sp1m_lp", "circ1024", "circ16384"]
# row-sharded fixed problems (--shard): SURVEY 8(e)
SHARD = {"cfg4": "cfg4", "cfg5b": "cfg5b"}
# the paper's circular forward table (FFT size = input length, B=64, H=768)
for _n, _b in ((512, 64), (1024, 64), (4096, 64), (16384, 64), (65536, 64), (1 << 18, 16), (1 << 20, 4),
               (1 << 22, 1)):
    WORKLOADS[f"circ{_n}"] = _wl(f"circular fp16 conv (fft_size = N) B*H={_b * 768} N={_n}", _b, 768, _n,
                                 causal=False)

METRIC = "fused FFT-conv sequences/s & % HBM/tensor roofline, N=256–4M, at 1/2/4/8 B200"
# paper's padded (causal) H100 rows for the same workload, another
# machine: context only.  cfg2 = gated FFT-2K row 0.59 ms.
PAPER_SEQ_S = {"cfg2": 49152 / 0.59e-3}
# circular table rows (FlashFFTConv ms on H100 for 49,152 rows)
for _n, _ms in ((512, 0.15), (1024, 0.24), (4096, 1.37), (16384, 9.27), (65536, 67.96), (1 << 18, 308.48),
                (1 << 20, 1492.84), (1 << 22, 7586.96)):
    PAPER_SEQ_S[f"circ{_n}"] = 49152 / (_ms * 1e-3)


def sparsity_spec(kind, fft):
    if kind is None:
        return None
    if kind == "rows75":  # keep outer rows {0, 1, L0/2, L0-1} of the multipass layout
        L0 = fft // 2048
        keep = np.zeros(L0, bool)
        keep[[0, 1, L0 // 2, L0 - 1]] = True
        return ([2048, L0], [np.ones(2048, bool), keep])
    if kind == "lowpass8":  # keep f < L/8 (slowest digit of [16, L/16] < 2); Hermitian closure adds f > 7L/8
        dims = [16, fft // 16]
        return (dims, [np.arange(16) < 2, np.ones(fft // 16, bool)])
    if kind.startswith("paper:"):  # tab:sparsity_fraction pattern: trailing a,b,c,d zeroed on 32x32x32x64
        z = [int(x) for x in kind[6:].split(",")]
        dims = [32, 32, 32, 64]
        assert fft == int(np.prod(dims))
        return (dims, [np.arange(d) < d - a for d, a in zip(dims, z)])
    raise ValueError(kind)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), tc=float(d["bf16_tflops"]), src="measured")
    return dict(hbm=6650.0, tc=1590.0, src="fallback")


class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.002):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self.period = period

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        rs = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": rs, "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU oracle
_ORACLE_INPUTS = {}


def _oracle_inputs(wl, Bs, Hs):
    """Seeded inputs of a Bs x Hs sample of the workload (generated once per
    shape; generation is never timed)."""
    key = (wl["name"], Bs, Hs)
    if key not in _ORACLE_INPUTS:
        import synth
        from oracle import oracle as orc
        H, N, K = wl["H"], wl["N"], wl["K"]
        k = synth.decay_filters(0, Hs, K).astype(np.float32).astype(np.float64)
        rows = np.array([b * H + h for b in range(Bs) for h in range(Hs)])
        q = lambda name: synth.quantize(synth.normal(0, synth.TENSOR_IDS[name], rows, N).reshape(Bs, Hs, N),
                                        wl["dtype"])
        kw = dict(w=q("w"), v=q("v")) if wl["gated"] else {}
        mask = None
        if wl["sparse"]:
            dims, keeps = sparsity_spec(wl["sparse"], wl["fft"])
            mask = orc.frequency_mask(dims, keeps)
        _ORACLE_INPUTS.clear()  # keep one sample resident
        _ORACLE_INPUTS[key] = (q("u"), k, kw, mask, q("dy") if wl["bwd"] else None)
    return _ORACLE_INPUTS[key]


def _oracle_sample(wl, Bs, rows=None):
    """Run the fp64 oracle on Bs x (rows or H) rows of the workload; seconds."""
    from oracle import oracle as orc
    Hs = wl["H"] if rows is None else rows
    u, k, kw, mask, dy = _oracle_inputs(wl, Bs, Hs)
    t = time.perf_counter()
    orc.conv_fwd(u, k, causal=wl["causal"], mask=mask, **kw)
    if wl["bwd"]:
        orc.conv_bwd(dy, u, k, causal=wl["causal"], mask=mask, **kw)
    return time.perf_counter() - t


def oracle_rows_per_s(wl, target_s=8.0):
    """The fp64 oracle as it stands, on a bounded sample of the workload's
    rows, on this host's cores.  Returns (rows/s, cores, sample text, seconds, Bs, Hs)."""
    from oracle import oracle as orc
    H, N = wl["H"], wl["N"]
    h0 = max(1, min(H, (1 << 20) // N))  # calibration: ~1M samples (per-call overhead amortised)
    dt = _oracle_sample(wl, 1, h0)
    rows = max(1.0, target_s / max(dt / h0, 1e-6))  # rows that fit the per-step budget
    if rows < H:
        Bs, Hs = 1, max(1, int(rows))
    else:
        Bs, Hs = max(1, min(wl["B"], int(rows / H))), H
    if (Bs, Hs) != (1, h0):
        dt = _oracle_sample(wl, Bs, Hs)
    what = ("gated " if wl["gated"] else "") + ("fwd+bwd" if wl["bwd"] else "fwd")
    sample = f"{Bs}x{Hs} rows of N={N} ({what} causal conv + k_f per head), fp64 oracle, {orc.num_threads()} threads"
    return Bs * Hs / dt, orc.num_threads(), sample, dt, Bs, Hs


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    # each step a bounded sample sized so the whole run stays around two minutes
    per_step = min(20.0, max(0.02, 120.0 / max(1, args.steps + min(args.warmup, 1))))
    rate, cores, sample, dt, Bs, Hs = oracle_rows_per_s(wl, target_s=per_step)
    for _ in range(min(args.warmup, 1)):
        _oracle_sample(wl, Bs, Hs)
    ts = [_oracle_sample(wl, Bs, Hs) for _ in range(args.steps)]
    step = statistics.mean(ts)
    value = Bs * Hs / step
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sequences/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"] + f" -- bounded sample of {Bs}x{Hs} rows per step",
                   "B": Bs, "H": Hs, "N": wl["N"], "fft_size": wl["fft"]},
        "cpu_baseline": {"value": value, "unit": "sequences/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "sequences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- GPU arm
def algorithmic_bytes(wl, H_L8):
    B, H, N = wl["B"], wl["H"], wl["N"]
    el = B * H * N * 2  # one (B, H, N) tensor of 16-bit I/O
    fwd = el * (4 if wl["gated"] else 2) + H_L8
    if not wl["bwd"]:
        return fwd
    bwd = el * (7 if wl["gated"] else 3) + H_L8 + H * wl["K"] * 4
    return fwd + bwd


def min_tensor_flops_per_row(wl):
    """the method's own minimum tensor-core work per row --
    Monarch stages over the packed complex length M = L/2, 8 M M_i real flops
    per stage and direction (fwd + inv), the causal halves of the first
    forward and last inverse stage removed, minimised over p <= 4 orders with
    factors >= 8 (powers of two).  Backward: x1.5 (plain) or x2 (gated)."""
    import itertools
    M = wl["fft"] // 2
    lg = M.bit_length() - 1
    best = None
    for p in (2, 3, 4):
        for parts in itertools.product(range(3, lg + 1), repeat=p):
            if sum(parts) != lg:
                continue
            f = [1 << e for e in parts]
            fl = sum(8 * M * m for m in f) * 2
            if wl["causal"]:
                fl -= 8 * M * f[0] // 2 * 2  # first forward stage (half K) and last inverse (half outputs)
            best = fl if best is None else min(best, fl)
    if best is None:
        return 0.0
    rows_per_row = 1.0
    if wl["causal"] and wl["fft"] < 2 * wl["N"]:  # partial: N / C windows of length L per row
        rows_per_row = wl["N"] / (wl["fft"] // 2)
    fl = best * rows_per_row  # M = L/2 is already the per-row packed length
    if wl["bwd"]:
        fl *= 3.0 if wl["gated"] else 2.5  # fwd + bwd (x2 gated, x1.5 plain)
    return fl


# ----------------------------------------------------------------- B1 baseline
def torch_fft_baseline(wl, u, w, v, k, dy, steps, mask=None):
    """cuFFT + PyTorch, the Hyena reference fftconv (inputs
    upcast to fp32, rfft of the padded rows, pointwise k_f, irfft, crop,
    gate); the filter FFT is inside the step as in ours; backward workloads
    through autograd.  Returns (ms per step, peak extra device bytes)."""
    import torch
    L, N = wl["fft"], wl["N"]
    if wl["causal"] and L < 2 * N:
        L = 2 * N  # partial conv: the plain FFT conv with the truncated filter
    m = None if mask is None else torch.tensor(mask[: L // 2 + 1], dtype=torch.float32, device=u.device)

    def step():
        rg = wl["bwd"]
        kk = k.detach().requires_grad_(rg)
        uu = u.float().requires_grad_(rg)
        g = uu * w.float().requires_grad_(rg) if w is not None else uu
        kf = torch.fft.rfft(kk, n=L)
        if m is not None:
            kf = kf * m
        y = torch.fft.irfft(torch.fft.rfft(g, n=L) * kf, n=L)[..., :N]
        if v is not None:
            y = y * v.float().requires_grad_(rg)
        if wl["bwd"]:
            y.backward(dy.float())
        return y.to(u.dtype)

    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    step()
    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, torch.cuda.max_memory_allocated() - base


class Run:
    """One workload set up on one device: plan, resident inputs, k_f buffer,
    workspaces and the conv closure (fwd [+ bwd]) through the C ABI."""

    def __init__(self, wl, dev, rank=0, h_range=None, seed_rank=0):
        import torch

        import synth
        from paper_2311_05908_b200 import FFTConvPlan, _abi
        from paper_2311_05908_b200.fftconv import _ptr, _stream
        self.wl, self.dev = wl, dev
        B, H, N, K, L = wl["B"], wl["H"], wl["N"], wl["K"], wl["fft"]
        h0, h1 = h_range if h_range is not None else (0, H)
        self.Hl = Hl = h1 - h0
        self.tdt = tdt = {"f16": torch.float16, "bf16": torch.bfloat16}[wl["dtype"]]
        self.plan = plan = FFTConvPlan(N, fft_size=L, dtype=tdt, causal=wl["causal"], device=dev,
                                       sparsity=sparsity_spec(wl["sparse"], L))

        def sig(name):
            if h_range is None:  # this rank's own B x H rows (weak scaling)
                return synth.signal_torch(0, name, B, H, N, dev, tdt, row0=rank * B * H)
            # head shard of the global problem: rows b * H + h, h in [h0, h1)
            return torch.cat([synth.signal_torch(0, name, 1, Hl, N, dev, tdt, row0=b * H + h0) for b in range(B)])

        self.u = sig("u")
        self.w = sig("w") if wl["gated"] else None
        self.v = sig("v") if wl["gated"] else None
        self.dy = sig("dy") if wl["bwd"] else None
        kfull = synth.decay_filters_torch(seed_rank, H, K, dev)
        self.k = kfull[h0:h1].contiguous()
        self.y = torch.empty_like(self.u)
        self.ws_f = plan.workspace(B, Hl, device=dev)
        self.ws_b = plan.workspace(B, Hl, for_bwd=True, device=dev) if wl["bwd"] else None
        self.grads = None
        if wl["bwd"]:
            u = self.u
            self.grads = dict(du=torch.empty_like(u), dw=torch.empty_like(u) if self.w is not None else None,
                              dv=torch.empty_like(u) if self.v is not None else None,
                              dk=torch.empty(Hl, K, dtype=torch.float32, device=dev))
        self.kfb = plan.kf_buffer(Hl, dev)  # reused every step (N = 4M: 64 MB of fp32 k_f per head)
        self._abi, self._ptr, self._stream = _abi, _ptr, _stream

    def kf(self, k=None):
        return self.plan.precompute_kf(self.k if k is None else k, out=self.kfb)

    def conv(self, kf, uu=None, ww=None, vv=None, out=None):
        wl, plan, B, K = self.wl, self.plan, self.wl["B"], self.wl["K"]
        uu = self.u if uu is None else uu
        ww = self.w if ww is None else ww
        vv = self.v if vv is None else vv
        out = self.y if out is None else out
        if wl["gated"]:
            plan.gated_fwd(uu, ww, vv, kf, out=out, workspace=self.ws_f)
        else:
            plan.fwd(uu, kf, out=out, workspace=self.ws_f)
        if wl["bwd"]:
            g, p = self.grads, self._ptr
            self._abi.check(self._abi.lib().fftconv_bwd(
                plan._h, p(self.dy), p(uu), p(ww), p(vv), p(kf), p(g["du"]), p(g["dw"]), p(g["dv"]), p(g["dk"]),
                B, self.Hl, K, p(self.ws_b), self._stream(self.dev)))

    def time(self, steps, warmup, world=1, clock_index=0):
        """W untimed steps, then S timed steps of precompute_kf + conv with
        CUDA events on the launching stream; returns (step ms, conv ms,
        launches, clocks), each the max over ranks."""
        import torch
        import torch.distributed as dist
        from paper_2311_05908_b200 import launch_count_reset
        for _ in range(warmup):
            self.conv(self.kf())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev_s = torch.cuda.Event(enable_timing=True)
        ev_e = torch.cuda.Event(enable_timing=True)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        launch_count_reset()
        with ClockSampler(clock_index) as clk:
            torch.cuda.synchronize()
            ev_s.record()
            for i in range(steps):
                kf = self.kf()
                ev[i][0].record()
                self.conv(kf)
                ev[i][1].record()
            ev_e.record()
            torch.cuda.synchronize()
        launches = launch_count_reset()
        if world > 1:
            dist.barrier()
        total_ms = ev_s.elapsed_time(ev_e)
        conv_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
        if world > 1:
            t = torch.tensor([total_ms, conv_ms], device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms, conv_ms = t.tolist()
        return total_ms / steps, conv_ms, launches, clk.summary()

    def release(self):
        for name in ("u", "w", "v", "dy", "y", "ws_f", "ws_b", "grads", "kfb", "k", "plan"):
            setattr(self, name, None)


def roofline_of(wl, conv_ms, H_local, peaks, traffic=None):
    """Algorithmic bytes of one conv call (16-bit I/O tensors +
    fp32 k_f of the call's heads) over its measured time, and the governing
    roofline (max of HBM bytes and the method's minimum tensor flops)."""
    w2 = dict(wl)
    w2["H"] = H_local
    bytes_per_call = algorithmic_bytes(w2, H_local * wl["fft"] * 8)
    achieved = bytes_per_call / (conv_ms * 1e-3) / 1e9
    tflops = min_tensor_flops_per_row(wl) * wl["B"] * H_local
    t_hbm = bytes_per_call / (peaks["hbm"] * 1e9)
    t_tc = tflops / (peaks["tc"] * 1e12)
    governing = {"bound": "hbm" if t_hbm >= t_tc else "tensor", "frac": max(t_hbm, t_tc) / (conv_ms * 1e-3),
                 "min_tensor_flops_per_call": tflops, "tensor_peak_tflops": peaks["tc"]}
    return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm"], "unit": "GB/s",
            "frac": achieved / peaks["hbm"], "traffic": traffic, "kernel_ms": conv_ms,
            "algorithmic_bytes_per_launch": bytes_per_call, "peak_source": peaks["src"], "governing": governing}


def _traffic(name):
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            return json.load(open(prof)).get(name, {}).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_sweep(names, dev, peaks, steps_small, steps_big, warmup):
    """Every regime of the metric: per point seq/s of the step,
    conv ms, roofline fraction on the same measured peak, clocks.  Launched
    one after another on this GPU, each with its own inputs (> L2)."""
    import torch
    out = {}
    for name in names:
        wl = WORKLOADS[name]
        try:
            r = Run(wl, dev)
            S = steps_small if wl["B"] * wl["H"] * wl["N"] <= (1 << 26) else steps_big
            step_ms, conv_ms, launches, clocks = r.time(S, warmup, clock_index=dev.index or 0)
            rf = roofline_of(wl, conv_ms, wl["H"], peaks, _traffic(name))
            out[name] = {"workload": wl["name"], "seq_per_s": wl["B"] * wl["H"] / (step_ms * 1e-3),
                         "ms_per_step": step_ms, "conv_ms": conv_ms, "frac": rf["frac"],
                         "governing": rf["governing"]["bound"], "governing_frac": rf["governing"]["frac"],
                         "algorithmic_bytes": rf["algorithmic_bytes_per_launch"], "traffic": rf["traffic"],
                         "regime": {1: "fused", 2: "partial", 3: "multipass"}[r.plan.info.regime],
                         "skip_fraction": r.plan.info.skip_fraction if wl["sparse"] else None,
                         "steps": S, "gpu_launches": launches, "clocks": clocks}
            if name in PAPER_SEQ_S:
                out[name]["paper_h100_seq_per_s"] = PAPER_SEQ_S[name]
            r.release()
            del r
        except torch.OutOfMemoryError as e:
            out[name] = {"unavailable": f"out of memory: {e}"[:200]}
        torch.cuda.empty_cache()
    return out


def run_shard(args, wl, dev, rank, world):
    """one FIXED problem head-sharded over WORLD_SIZE ranks
    (strong scaling; rows independent).  compute-only: every rank
    convolves its resident shard; end-to-end: rank 0 holds the full (B, H,
    N) tensors, NCCL scatters head shards (paper_2311_05908_b200.dist), each
    rank convolves, NCCL gathers y back to rank 0.  Both timed on the device
    with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2311_05908_b200.dist import gather_heads, head_shard, scatter_heads
    B, H, N = wl["B"], wl["H"], wl["N"]
    h0, h1 = head_shard(H, rank, world)
    r = Run(wl, dev, h_range=(h0, h1))
    step_ms, conv_ms, launches, clocks = r.time(args.steps, args.warmup, world, dev.index or 0)
    # end to end from rank 0's device tensors
    full = {}
    if rank == 0:
        import synth
        for name in ("u", "w", "v"):
            if name == "u" or wl["gated"]:
                full[name] = synth.signal_torch(0, name, B, H, N, dev, r.tdt)
    def e2e_once():
        parts = {name: scatter_heads(full.get(name), H, (B, N), r.tdt, dev) for name in ("u", "w", "v")
                 if name == "u" or wl["gated"]}
        kf = r.kf()
        r.conv(kf, parts["u"], parts.get("w"), parts.get("v"), r.y)
        return gather_heads(r.y, H)
    for _ in range(2):
        e2e_once()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    E = max(3, min(args.steps, 10))
    e0.record()
    for _ in range(E):
        e2e_once()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / E], device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = e2e_ms.item()
    if rank == 0:
        peaks = load_peaks()
        rf = roofline_of(wl, conv_ms, h1 - h0, peaks)
        moved = B * H * N * 2 * ((3 if wl["gated"] else 1) + 1)
        out = {
            "metric": METRIC, "value": B * H / (step_ms * 1e-3), "unit": "sequences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": wl["name"] + f" -- fixed problem, heads sharded over {world} GPU(s)",
                       "B": B, "H": H, "N": N, "K": wl["K"], "fft_size": wl["fft"],
                       "heads_per_rank": [b - a for a, b in (head_shard(H, q, world) for q in range(world))],
                       "parallelism": f"head-sharded x{world}, NCCL scatter/gather only outside the conv"},
            "roofline": dict(rf, note="rank 0's shard (its heads, all B)"),
            "compute_only": {"value": B * H / (step_ms * 1e-3), "ms_per_step": step_ms, "conv_ms": conv_ms,
                             "note": "resident shards (inputs generated on each rank), precompute_kf + conv"},
            "e2e": {"value": B * H / (e2e_ms * 1e-3), "unit": "sequences/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0, "nccl_bytes_per_step": moved,
                    "path": "rank 0 device tensors -> NCCL scatter (u[, w, v]) -> conv -> NCCL gather (y)"},
            "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="fftconv", choices=["fftconv", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-torch-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the per-regime sweep object")
    ap.add_argument("--sweep", default=None, help="comma-separated sweep workloads (default: SWEEP)")
    ap.add_argument("--shard", default=None, choices=sorted(SHARD),
                    help="fixed problem head-sharded over WORLD_SIZE ranks (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.shard or args.workload]
    if args.steps is None:
        args.steps = 500 if wl["B"] * wl["H"] * wl["N"] <= (1 << 26) else 40

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1 or args.shard:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    if args.shard:
        run_shard(args, wl, dev, rank, world)
        dist.barrier()
        dist.destroy_process_group()
        return

    B, H, N, K, L = wl["B"], wl["H"], wl["N"], wl["K"], wl["fft"]
    run = Run(wl, dev, rank=rank, seed_rank=rank)
    plan, u, w, v, dy, k, y = run.plan, run.u, run.w, run.v, run.dy, run.k, run.y
    S = args.steps
    step_ms, conv_ms, launches, clocks = run.time(S, args.warmup, world, local_rank)
    value = world * B * H / (step_ms * 1e-3)

    # ---------------- end-to-end through the public API with pinned host buffers
    def pinned_copy(t):  # straight into pinned host memory (no pageable staging copy)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    hbuf = {name: pinned_copy(t) for name, t in (("u", u), ("w", w), ("v", v), ("dy", dy), ("k", k))
            if t is not None}
    rpc = max(1, B // 8)
    use_host_api = not wl["bwd"] and B >= 2
    dbuf = {name: torch.empty_like(t) for name, t in (("u", u), ("w", w), ("v", v), ("k", k))
            if t is not None and (name == "k" or not use_host_api)}
    hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
    h2d = sum(t.numel() * t.element_size() for t in hbuf.values())
    d2h = hy.numel() * hy.element_size()
    if wl["bwd"]:
        hdu = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
        d2h += hdu.numel() * hdu.element_size() + run.grads["dk"].numel() * 4

    # forward workloads with B >= 2 go through fftconv_fwd_host: batch chunks
    # streamed through a device staging buffer, copies overlapping the conv
    stage = plan.host_stage(H, rpc, wl["gated"], dev) if use_host_api else None

    def e2e_step():
        if use_host_api:
            dbuf["k"].copy_(hbuf["k"], non_blocking=True)
            kf = run.kf(dbuf["k"])
            plan.fwd_host(hbuf["u"], kf, w=hbuf.get("w"), v=hbuf.get("v"), out=hy, rows_per_chunk=rpc, stage=stage)
            return
        for name, t in dbuf.items():
            t.copy_(hbuf[name], non_blocking=True)
        if dy is not None:
            dy.copy_(hbuf["dy"], non_blocking=True)
        kf = run.kf(dbuf["k"])
        run.conv(kf, dbuf["u"], dbuf.get("w"), dbuf.get("v"), y)
        hy.copy_(y, non_blocking=True)
        if wl["bwd"]:
            hdu.copy_(run.grads["du"], non_blocking=True)

    E = max(3, args.e2e_steps) if args.e2e_steps > 0 else 0  # 0: no e2e leg (profiling runs)
    for _ in range(2 if E else 0):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(E):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / E if E else float("nan")
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    e2e_value = world * B * H / (e2e_ms * 1e-3)

    if rank == 0:
        peaks = load_peaks()
        rf = roofline_of(wl, conv_ms, H, peaks, _traffic(args.workload))
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            rate, cores, sample, _, _, _ = oracle_rows_per_s(wl)
            cpu = {"value": rate, "unit": "sequences/s", "cores": cores, "kind": "oracle", "sample": sample,
                   "cpu_model": _cpu_model()}
            try:  # the same oracle on one core
                from oracle import oracle as orc
                nt = orc.num_threads()
                orc.set_num_threads(1)
                r1, _, s1, _, _, _ = oracle_rows_per_s(wl, target_s=4.0)
                orc.set_num_threads(nt)
                cpu["one_core"] = {"value": r1, "unit": "sequences/s", "sample": s1}
            except Exception as e:  # pragma: no cover
                cpu["one_core"] = {"unavailable": str(e)[:200]}
        vs = PAPER_SEQ_S.get(args.workload)
        regime = {1: "fused", 2: "partial (overlap-save, multipass)", 3: "multipass"}[plan.info.regime]
        # device memory of this library for the step vs the cuFFT+PyTorch reference (NEXT-3)
        lib_bytes = run.kfb.numel() + (run.ws_f.numel() if run.ws_f is not None else 0) \
            + (run.ws_b.numel() if run.ws_b is not None else 0) + plan.info.table_bytes
        tb = None
        if not args.no_torch_baseline:
            spec = B * H * (max(L, 2 * N) // 2 + 1) * 8  # one complex64 spectrum of the batch
            free, _ = torch.cuda.mem_get_info(dev)
            if spec * (10 if wl["bwd"] else 6) < free:
                try:  # (sparse workloads: dense spectrum product, the mask multiply is the same cost)
                    ms_b, peak_b = torch_fft_baseline(wl, u, w, v, k, dy, min(S, 20))
                    tb = {"value": B * H / (ms_b * 1e-3), "unit": "sequences/s", "ms_per_step": ms_b,
                          "peak_extra_bytes": int(peak_b),
                          "kind": "torch.fft (cuFFT) fp32 Hyena-style fftconv" + (" + autograd bwd" if wl["bwd"] else ""),
                          "speedup_of_this": (B * H / (step_ms * 1e-3)) / (B * H / (ms_b * 1e-3))}
                except torch.OutOfMemoryError:
                    tb = {"value": None, "unavailable": "out of memory"}
            else:
                tb = {"value": None, "unavailable": "would not fit beside this run's buffers"}
        rf["kernel"] = ("conv call (fftconv_fwd_o2_kernel" + (" + multipass outer passes" if plan.info.regime != 1 else "")
                        + (" + bwd" if wl["bwd"] else "") + ")")
        rf["governing"]["note"] = ("fraction of the governing roofline (HBM bytes vs the method's minimum Monarch "
                                   "tensor flops, p <= 4, SURVEY 8(d))")
        out = {
            "metric": METRIC, "value": value, "unit": "sequences/s", "n_gpus": world, "steps": S,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": (value / vs) if vs else None,
            "vs_baseline_note": ("paper H100-SXM " + ("padded gated FFT-2K row (P:1144-1167)" if args.workload == "cfg2"
                                                       else "circular forward row (P:1072-1095)")
                                 + ", conv only there, k_f precompute included here; another machine: context only")
            if vs else None,
            "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": wl["name"], "B": B, "H": H, "N": N, "K": K, "fft_size": L, "gated": wl["gated"],
                       "causal": wl["causal"], "backward": wl["bwd"], "regime": regime,
                       "step": "precompute_kf + conv" + (" fwd+bwd" if wl["bwd"] else " fwd"),
                       "l2": f"inputs larger than L2 ({rf['algorithmic_bytes_per_launch'] / 1e6:.0f} MB per step)",
                       "parallelism": f"rows sharded, {world} GPU(s), no data-path collective"},
            "roofline": rf,
            "cpu_baseline": cpu,
            "cufft_baseline": tb,
            "memory": {"library_device_bytes": int(lib_bytes),
                       "note": "k_f + workspace(s) + plan tables; caller-owned, reused every step"},
            "e2e": None if not E else {"value": e2e_value, "unit": "sequences/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "path": (f"fftconv_fwd_host, {(B + rpc - 1) // rpc} chunks of {rpc} batch rows, copies overlapped"
                             if use_host_api else "device copies around fftconv calls")},
            "gpu_launches": launches,
            "clocks": clocks,
        }
    # ---------------- every regime of the metric, same run (rank 0's GPU; N=1 only)
    if world == 1 and not args.no_sweep:
        run.release()
        del run, plan, u, w, v, dy, k, y, hbuf, dbuf, stage
        torch.cuda.empty_cache()
        names = args.sweep.split(",") if args.sweep else SWEEP
        out["sweep"] = run_sweep(names, dev, load_peaks(), steps_small=30, steps_big=5, warmup=3)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


if __name__ == "__main__":
    main()
