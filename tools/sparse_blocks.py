"""How much of the paper's frequency-sparse patterns (tab:sparsity_fraction,
P:1045-1060, on the 2M-point grid 32x32x32x64 of P:1035) survives the
Hermitian closure m[f] = keep(f) | keep(L - f) (A13(iii)), and which Monarch
blocks of this library's N = 1M plan (f = k0 + 1024 f', f' = k2 + 64 k1;
inner rows = k0, stage-B groups = k2 / 32, stage-B column chunks = k1 / 8)
are entirely zero -- i.e. what a kernel could skip without changing y."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc

g = json.load(open(os.path.join(ROOT, "tests", "golden", "sparsity_fraction.json")))
dims = g["dims"]
L = int(np.prod(dims))
f = np.arange(L)
k0, fp = f % 1024, f // 1024
k2, k1 = fp % 64, fp // 64
print("| pattern (a,b,c,d) | S printed | keep(f) zero fraction | after closure | zero inner rows k0 | "
      "zero (k0, k2-group, k1-chunk) blocks | zero (k2-group, k1-chunk) blocks for all k0 |")
print("|---|---|---|---|---|---|---|")
for row in g["rows"]:
    keeps = orc.keep_masks_from_zero_counts(dims, row["zeroed"])
    kp = orc.keep_set(dims, keeps)
    m = orc.frequency_mask(dims, keeps) > 0
    rows_zero = 1 - np.mean([m[k0 == r].any() for r in range(1024)])
    blk = np.zeros((1024, 2, 4), bool)
    np.logical_or.at(blk, (k0, k2 // 32, k1 // 8), m)
    gk = blk.any(axis=0)
    print(f"| {tuple(row['zeroed'])} | {row['S_percent']} % | {1 - kp.mean():.4f} | {1 - m.mean():.4f} | "
          f"{rows_zero:.4f} | {1 - blk.mean():.4f} | {1 - gk.mean():.4f} |")
