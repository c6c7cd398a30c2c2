"""The parity bar every GPU test applies (BASELINE.json north_star):

* fp16 / bf16 I/O: rel-L2 <= 2e-3 AND max-abs <= 1e-2 * max|ref| against
  the fp64 oracle, on the compared set (whole tensors, or the sampled
  outputs of a full-size check);
* fp32 validation build: rel-L2 <= 1e-5 (and the same max-abs bar scaled by
  the rel-L2 ratio, 5e-5 * max|ref|).

Both sides must also be finite.  Test infrastructure only."""
import numpy as np

REL_L2 = 2e-3
MAX_ABS = 1e-2
REL_L2_F32 = 1e-5
MAX_ABS_F32 = 5e-5


def errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
    mx = float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)) if ref.size else 0.0
    return rel, mx


def assert_parity(got, ref, what="", rel_l2=REL_L2, max_abs=MAX_ABS):
    """fp16/bf16 bar; returns (rel-L2, max-abs / max|ref|)."""
    assert np.all(np.isfinite(got)), f"{what}: non-finite output"
    rel, mx = errors(got, ref)
    assert rel <= rel_l2 and mx <= max_abs, f"{what}: rel-L2 {rel:.3e} (<= {rel_l2}), max-abs {mx:.3e} (<= {max_abs})"
    return rel, mx


def assert_parity_f32(got, ref, what=""):
    return assert_parity(got, ref, what, REL_L2_F32, MAX_ABS_F32)
