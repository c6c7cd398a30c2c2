"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle-side tests and the CUDA-side tests and
bench; it holds none of the method's arithmetic (no transforms, no
convolution), only a counter-based random generator and the input recipes
stated in DESIGN.md ("Input recipe"):

* u, w, v, dy ~ N(0, 1), cast to the I/O dtype;
* Hyena-like decaying filters k[h, t] = N(0,1) * exp(-lambda_h t / K) /
  sqrt(sum_t exp(-2 lambda_h t / K)), lambda_h log-spaced in [0.5, 50] over
  heads, so |y| = O(1);
* a flat N(0, 1/K) filter;
* "DNA-like" piecewise-constant rows (HyenaDNA).

Every value is a pure function of (seed, tensor id, row, position), so any
shard of rows can be generated independently (counter-based, splitmix64).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_C_SEED = np.uint64(0x9E3779B97F4A7C15)
_C_TENSOR = np.uint64(0xD1B54A32D192ED03)
_C_ROW = np.uint64(0x8CB92BA72F3D8DD7)
_C_ALT = np.uint64(0xA0761D6478BD642F)

TENSOR_IDS = {"u": 1, "w": 2, "v": 3, "dy": 4, "k": 5, "aux": 6}


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def _keys(seed: int, tensor: int, rows: np.ndarray, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = (np.uint64(seed) * _C_SEED + np.uint64(tensor) * _C_TENSOR)
        r = rows.astype(np.uint64)[:, None] * _C_ROW
        return base + r + np.arange(n, dtype=np.uint64)[None, :]


def uniform(seed: int, tensor: int, rows, n: int) -> np.ndarray:
    """U(0,1] array of shape (len(rows), n)."""
    rows = np.asarray(rows, dtype=np.int64)
    h = _mix(_keys(seed, tensor, rows, n))
    return ((h >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def normal(seed: int, tensor: int, rows, n: int) -> np.ndarray:
    """N(0,1) array of shape (len(rows), n) via Box-Muller on two hashes."""
    rows = np.asarray(rows, dtype=np.int64)
    k = _keys(seed, tensor, rows, n)
    with np.errstate(over="ignore"):
        h1 = _mix(k)
        h2 = _mix(k ^ _C_ALT)
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
    u2 = (h2 >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def signal(seed: int, name: str, B: int, H: int, N: int, row0: int = 0,
           nrows: int | None = None) -> np.ndarray:
    """(B, H, N) N(0,1) fp64 tensor (or a contiguous slice of its B*H rows
    starting at row0 when nrows is given; rows are b*H + h)."""
    total = B * H
    nrows = total - row0 if nrows is None else nrows
    rows = np.arange(row0, row0 + nrows)
    x = normal(seed, TENSOR_IDS[name], rows, N)
    return x.reshape(B, H, N) if (row0 == 0 and nrows == total) else x


def decay_filters(seed: int, H: int, K: int, lam_lo: float = 0.5,
                  lam_hi: float = 50.0) -> np.ndarray:
    """(H, K) fp64 Hyena-like exponentially decaying filters, unit L2 norm."""
    lam = np.exp(np.linspace(np.log(lam_lo), np.log(lam_hi), max(H, 1)))[:H]
    t = np.arange(K, dtype=np.float64)
    env = np.exp(-lam[:, None] * t[None, :] / max(K, 1))
    z = normal(seed, TENSOR_IDS["k"], np.arange(H), K)
    k = z * env
    return k / np.sqrt((env ** 2).sum(axis=1, keepdims=True))


def flat_filters(seed: int, H: int, K: int) -> np.ndarray:
    """(H, K) N(0, 1/K) filters."""
    return normal(seed, TENSOR_IDS["k"], np.arange(H), K) / np.sqrt(max(K, 1))


def dna_like(seed: int, B: int, H: int, N: int, run: int = 64) -> np.ndarray:
    """Piecewise-constant rows over 4 embedding levels (single-nucleotide
    tokens mimic; HyenaDNA workload P:744)."""
    levels = normal(seed, TENSOR_IDS["aux"], np.arange(H), 4)  # (H, 4)
    nrun = (N + run - 1) // run
    pick = (uniform(seed, TENSOR_IDS["aux"] + 100, np.arange(B * H), nrun) * 4).astype(np.int64)
    pick = np.minimum(pick, 3)
    lv = levels[np.arange(B * H) % H]
    vals = np.take_along_axis(lv, pick, axis=1)
    return np.repeat(vals, run, axis=1)[:, :N].reshape(B, H, N)


def quantize(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round to the I/O dtype ('f16', 'bf16', 'f32') and return as fp64, so
    the oracle consumes exactly the values the GPU consumes."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        f = x.astype(np.float32)
        b = f.view(np.uint32).astype(np.uint64)
        # round-to-nearest-even on the upper 16 bits
        lsb = (b >> np.uint64(16)) & np.uint64(1)
        b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
        return b.astype(np.uint32).view(np.float32).astype(np.float64)
    raise ValueError(dtype)


# --------------------------------------------------------------------------
# same generator on a torch device (for large bench inputs)
# --------------------------------------------------------------------------
def _to_i64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def _mix_t(x):
    import torch
    m30 = (1 << 34) - 1
    m27 = (1 << 37) - 1
    m31 = (1 << 33) - 1
    x = x ^ ((x >> 30) & m30)
    x = x * _to_i64(0xBF58476D1CE4E5B9)
    x = x ^ ((x >> 27) & m27)
    x = x * _to_i64(0x94D049BB133111EB)
    x = x ^ ((x >> 31) & m31)
    return x


def normal_torch(seed: int, tensor: int, row0: int, nrows: int, n: int, device, chunk_elems: int = 1 << 25):
    """Same counter-based N(0,1) stream as normal(), generated with int64
    torch ops on `device` (values agree with numpy up to the last bits of
    log/cos); returns float32 (nrows, n)."""
    import torch
    out = torch.empty(nrows, n, dtype=torch.float32, device=device)
    base = _to_i64((seed * 0x9E3779B97F4A7C15 + tensor * 0xD1B54A32D192ED03) % (1 << 64))
    cr = _to_i64(0x8CB92BA72F3D8DD7)
    alt = _to_i64(0xA0761D6478BD642F)
    cols_per = max(1, min(n, chunk_elems))
    rows_per = max(1, chunk_elems // n)
    for r0 in range(0, nrows, rows_per):
        r1 = min(nrows, r0 + rows_per)
        rows = torch.arange(row0 + r0, row0 + r1, dtype=torch.int64, device=device)
        for c0 in range(0, n, cols_per):
            c1 = min(n, c0 + cols_per)
            cols = torch.arange(c0, c1, dtype=torch.int64, device=device)
            k = base + rows[:, None] * cr + cols[None, :]
            h1 = _mix_t(k)
            h2 = _mix_t(k ^ alt)
            u1 = (((h1 >> 11) & ((1 << 53) - 1)).double() + 1.0) * (1.0 / 9007199254740992.0)
            u2 = ((h2 >> 11) & ((1 << 53) - 1)).double() * (1.0 / 9007199254740992.0)
            out[r0:r1, c0:c1] = (torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * np.pi * u2)).float()
    return out


def signal_torch(seed: int, name: str, B: int, H: int, N: int, device, dtype, row0: int = 0):
    """(B, H, N) tensor of the given torch dtype on device; rows row0.. of the
    global (b*H + h) numbering (row0 lets ranks generate their own shard)."""
    import torch
    out = torch.empty(B * H, N, dtype=dtype, device=device)
    step = max(1, (1 << 27) // N)  # rows per fp32 staging chunk
    for r in range(0, B * H, step):
        r1 = min(B * H, r + step)
        out[r:r1] = normal_torch(seed, TENSOR_IDS[name], row0 + r, r1 - r, N, device).to(dtype)
    return out.reshape(B, H, N)


def decay_filters_torch(seed: int, H: int, K: int, device, lam_lo: float = 0.5, lam_hi: float = 50.0):
    """decay_filters() generated on `device` (float32 (H, K)); same stream and
    recipe, for workloads whose filters do not fit host memory comfortably."""
    import torch
    out = normal_torch(seed, TENSOR_IDS["k"], 0, H, K, device)
    lam = np.exp(np.linspace(np.log(lam_lo), np.log(lam_hi), max(H, 1)))[:H]
    step = max(1, (1 << 26) // max(K, 1))
    for h0 in range(0, H, step):
        h1 = min(H, h0 + step)
        t = torch.arange(K, dtype=torch.float64, device=device)
        lt = torch.tensor(lam[h0:h1], dtype=torch.float64, device=device)
        env = torch.exp(-lt[:, None] * t[None, :] / max(K, 1))
        nrm = torch.sqrt((env ** 2).sum(dim=1, keepdim=True))
        out[h0:h1] = (out[h0:h1].double() * env / nrm).float()
    return out
