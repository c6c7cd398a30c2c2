"""Prints the fp32 validation build's rel-L2 against the fp64 oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_f32 as t
for N, causal, gated, kw in ((1024, True, True, {}), (2048, False, True, {}), (8192, True, True, {}),
                             (16384, True, False, {}), (16384, True, False, dict(fft_size=4096, K=1500))):
    rel, plan = t._run(N, causal, gated, B=5, H=3, seed=40, **kw)
    print(f"fp32 N={N} causal={causal} gated={gated} {kw} regime={plan.info.regime} rel-L2={rel:.2e}")
