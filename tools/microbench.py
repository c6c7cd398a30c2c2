"""Experiment: TMEM read throughput and back-to-back tcgen05.mma cost
(selftest library microbenchmarks)."""
import ctypes, os
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2311_05908_b200", "libfftconv_selftest.so"))
torch.zeros(1, device="cuda")
out = np.zeros(4, dtype=np.int64)
for nw in (1, 4, 8, 16):
    it = 1000
    lib.fcst_tmem_ld_bench(it, nw, out.ctypes.data_as(ctypes.c_void_p))
    byts = nw * it * 32 * 32 * 4
    print(f"tmem ld: warps {nw:2d} cycles {out[0]}  bytes/cycle {byts / out[0]:.1f}")
for ts in (0, 1):
    for N in (32, 64, 96, 128, 192, 256):
        for n in (8, 64):
            lib.fcst_mma_rate(n, N, ts, out.ctypes.data_as(ctypes.c_void_p))
            print(f"mma {'ts' if ts else 'ss'} N={N:3d} n={n:3d}: issue {out[2]:6d} done {out[3]:6d} cyc/mma {out[3]/n:6.1f}")
for M in (64, 128):
    for N in (64, 128, 256):
        lib.fcst_mma_rate_m(64, M, N, 0, out.ctypes.data_as(ctypes.c_void_p))
        print(f"mma ss M={M} N={N:3d} n= 64: issue {out[2]:6d} done {out[3]:6d} cyc/mma {out[3]/64:6.1f}")
