"""Tolerance model of the FP8 forward's parity test (test infrastructure, not oracle).

DESIGN.md R25 fixes the kernel contract: S = Q K^T is exact, the un-normalised
probabilities P~_ij = exp(S_ij - m~_i) are rounded to E4M3 (RN, satfinite) before the
P~V product, l sums the fp32 P~, and the running max m~_i used in the exponent never
trails the row's true max m_i by more than 8 in log2 units (R19), i.e. P~ <= 2^8.
From that contract alone, per output element (i, c):

  * normal E4M3 range: |round(x) - x| <= 2^-4 |x|, so the normalised error is at most
    2^-4 * sum_j P_ij |V_jc|;
  * subnormal P~ (< 2^-6): |round(x) - x| <= 2^-10 absolute, divided by
    l~_i = sum_j exp(S_ij - m~_i) >= l_i = sum_j exp(S_ij - m_i) (m~_i <= m_i), so at
    most 2^-10 / l_i * sum_{j visible} |V_jc|.

The plain-definition values P, l come from the oracle; only the bound lives here.
"""
import numpy as np

from oracle import ref_attention as R


def fp8_pv_error_bound(q, k, v, scale: float, causal: bool) -> np.ndarray:
    """[N, d] per-element bound on |O_kernel - O| added by the E4M3 rounding of P~ (one head)."""
    v = np.abs(np.asarray(v, dtype=np.float64))
    s = R.scores(q, k, scale, causal)
    p, m, ell = R.softmax_rows(s)
    visible = np.isfinite(s).astype(np.float64)
    return 2.0 ** -4 * (p @ v) + (2.0 ** -10 / ell)[:, None] * (visible @ v)
