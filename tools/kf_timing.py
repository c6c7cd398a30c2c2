"""Experiment: warm timings of the cfg2 step parts (CUDA events over 200
back-to-back calls): k_f precompute alone, the conv alone, both alternating."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05908_b200 import FFTConvPlan

B, H, N = 64, 768, 1024
dev = torch.device("cuda")
plan = FFTConvPlan(N, 2 * N, torch.float16, causal=True)
k = torch.randn(H, N, device=dev)
u = torch.randn(B, H, N, device=dev, dtype=torch.float16)
w, v = torch.randn_like(u), torch.randn_like(u)
kf = plan.precompute_kf(k)
y = torch.empty_like(u)
def t(fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
print("precompute_kf us", t(lambda: plan.precompute_kf(k, out=kf)))
print("conv us", t(lambda: plan.gated_fwd(u, w, v, kf, out=y)))
print("both us", t(lambda: (plan.precompute_kf(k, out=kf), plan.gated_fwd(u, w, v, kf, out=y))))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): plan.precompute_kf(k, out=kf); plan.gated_fwd(u, w, v, kf, out=y)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    plan.precompute_kf(k, out=kf); plan.gated_fwd(u, w, v, kf, out=y)
print("graph both us", t(lambda: g.replay()))
