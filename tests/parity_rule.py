"""The parity tolerance rule, shared by the GPU
parity tests and smoke().

The oracle computes in fp64 and also returns `mag`, the absolute-value forward
(Σ|terms| carried through every linear stage) — the natural scale of
floating-point error for each output element.

  fp32 path  (FFMA FC, FFMA GRU):   |gpu - ref| <= 1e-5 * max(|ref|, mag * 2^-10)
                                    elementwise (verbatim)
  tf32 path  (tcgen05 kind::tf32):  |gpu - ref| <= 2^-10 * mag elementwise
                                    (both MMA operands are rounded to a 10-bit
                                    mantissa, so one product's error is at most
                                    2 * 2^-11 * |w||x|: Σ over a dot is 2^-10 *
                                    Σ|terms|), and normwise
                                    max|d| / max|ref| <= 5e-3
  bf16 path (RS_FC_BF16, labelled   |gpu - ref| <= 2^-5 * mag elementwise
  lower-precision variant):         (bf16 operands: unit roundoff 2^-8, so a
                                    product is within 2^-7 |w||x|; activations
                                    are re-rounded between layers; up to 4
                                    layers) and normwise max|d|/max|ref| <= 5e-2
                                    (measured: <= 1.5e-5*mag elementwise;
                                    normwise 0.002-0.005 at 200 items, 0.033
                                    for a single near-zero logit at S = 1)
  SLS pooled sums:                  bit-identical to the oracle's canonical
                                    fp32 summation order
  DIN attention-pooled sums         Σ_l a_l e_l over L lookups accumulated in
  (pooled output of AttentionFC):   fp32: the SURVEY rule, or Higham's bound
                                    for an L-term fp32 sum, |d| <= L * 2^-24 *
                                    Σ|terms| (γ_L), whichever is larger — the
                                    SURVEY rule alone is below what any L=200
                                    fp32 summation order can guarantee
  GRU/AUGRU hidden state (pooled    |h| < 1 (a convex mix of tanh outputs), so
  output of AttentionRNN):          the scale is 1: |d| <= 1e-5 (fp32 FFMA
                                    recurrence), |d| <= 1e-2 and normwise
                                    <= 5e-3 (tf32 tensor-core recurrence)
"""
import numpy as np

FP32 = "fp32"
TF32 = "tf32"
BF16 = "bf16"
TWO_M10 = 2.0 ** -10


def excess(got, ref, mag, path):
    """max over elements of |gpu-ref| / bound: <= 1 passes the rule."""
    d = np.abs(np.asarray(got, dtype=np.float64) - ref)
    if path == FP32:
        bound = 1e-5 * np.maximum(np.abs(ref), mag * TWO_M10)
    elif path == BF16:
        bound = 2.0 ** -5 * mag
    else:
        bound = TWO_M10 * mag
    return float(np.max(d / np.maximum(bound, 1e-300)))


def normwise(got, ref):
    d = np.abs(np.asarray(got, dtype=np.float64) - ref)
    return float(np.max(d) / max(float(np.max(np.abs(ref))), 1e-300))


def assert_close(got, ref, mag, path, what=""):
    x = excess(got, ref, mag, path)
    assert x <= 1.0, f"{what}: {path} rule exceeded by {x:.3g}x"
    if path in (TF32, BF16):
        nw = normwise(got, ref)
        lim = 5e-3 if path == TF32 else 5e-2
        assert nw <= lim, f"{what}: {path} normwise {nw:.3g} > {lim}"
    return x


def assert_attention_pooled(got, ref, mag, L, what=""):
    d = np.abs(np.asarray(got, dtype=np.float64) - ref)
    bound = np.maximum(1e-5 * np.maximum(np.abs(ref), mag * TWO_M10), L * 2.0 ** -24 * mag)
    x = float(np.max(d / np.maximum(bound, 1e-300)))
    assert x <= 1.0, f"{what}: attention-pooled rule exceeded by {x:.3g}x"
    return x


def assert_gru_state(got, ref, path, what=""):
    d = float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)))
    lim = 1e-5 if path == FP32 else 1e-2
    assert d <= lim, f"{what}: GRU state |d| = {d:.3g} > {lim}"
    if path == TF32:
        assert normwise(got, ref) <= 5e-3
    return d
