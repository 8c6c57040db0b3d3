"""CPU fp64 oracle for the FlashAttention-2 hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2307_08691_b200``) never imports it, and it
imports nothing from the product path: the two share no code.

What it computes is the *plain definition* of exact softmax attention, not the
tiled algorithm: FlashAttention-2 is exact ("with no approximation", PAPER.md
P:16), so the oracle materialises S and P in full.

Citations are PAPER.md line numbers (P:n) and SPEC.md line numbers (S:n) in
``/root/reference``.  Readings of garbled or silent passages are listed in
DESIGN.md §3 ("Readings"); the ones used here are referenced as R<n>.

Conventions (R1, R2, R8, R10):
  * q, k, v, do are float arrays of shape [B, H, N, d] (or [N, d] for the
    per-head functions); they are upcast to float64 before any arithmetic.
  * ``scale`` multiplies QK^T before the softmax (P:160-162 footnote; read as
    1/sqrt(d) by default, R1).  The caller passes the exact value the kernel
    receives (a float32), and it is used as float64(float32(scale)).
  * causal: S_ij = -inf for j > i, top-left aligned, N_q = N_k;
    the *_general / *_varlen functions extend it bottom-right aligned to
    N_q != N_k (R22) with empty rows O = 0, L = -inf (R23).
  * L is the natural-log logsumexp of the *scaled* logits.

Pins: every function here is checked by ``tests/test_oracle.py`` against
values the paper/spec print, closed forms, invariants and finite differences
(DESIGN.md §4).  No function in this file is "parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "as_f64_scale",
    "scores",
    "softmax_rows",
    "forward_head",
    "forward",
    "softmax_backward_row",
    "backward_head",
    "backward",
    "rowsum_dO_O",
    "forward_rows",
    "backward_sampled_head",
    "naive_softmax_no_max",
    "forward_gqa",
    "backward_gqa",
    "scores_general",
    "softmax_rows_general",
    "forward_head_general",
    "backward_head_general",
    "forward_varlen",
    "backward_varlen",
]


def as_f64_scale(scale: float) -> float:
    """The exact softmax scale the kernel receives (a float32), as float64 (R1)."""
    return float(np.float32(scale))


# ---------------------------------------------------------------------------
# Forward: standard attention
# ---------------------------------------------------------------------------

def scores(q: np.ndarray, k: np.ndarray, scale: float, causal: bool) -> np.ndarray:
    """S = scale * Q K^T  (scale per footnote P:160-162),
    with S_ij = -inf for j > i when causal."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    s = as_f64_scale(scale) * (q @ k.T)
    if causal:
        n_q, n_k = s.shape
        if n_q != n_k:
            raise ValueError("causal attention is defined here for N_q == N_k only (R8)")
        s[np.triu_indices(n_q, k=1)] = -np.inf
    return s


def softmax_rows(s: np.ndarray):
    """Row-wise softmax of P:158 written out as in P:225-227:
    m_i = max_j S_ij, E = exp(S - m), l_i = sum_j E_ij, P = E / l.
    Returns (P, m, l)."""
    m = np.max(s, axis=1)
    e = np.exp(s - m[:, None])
    ell = np.sum(e, axis=1)
    p = e / ell[:, None]
    return p, m, ell


def forward_head(q, k, v, scale: float, causal: bool):
    """One (b, h) head.  O = softmax(S) V; L = m + log(l).

    Returns (O [N,d], L [N]) in float64."""
    v = np.asarray(v, dtype=np.float64)
    s = scores(q, k, scale, causal)
    p, m, ell = softmax_rows(s)
    o = p @ v
    lse = m + np.log(ell)
    return o, lse


def forward(q, k, v, scale: float, causal: bool):
    """Batched [B, H, N, d]: the same computation per head, in parallel over
    batch and heads.  Returns (O [B,H,N,d], L [B,H,N]) float64."""
    q = np.asarray(q)
    b, h, n, d = q.shape
    o = np.empty((b, h, n, d), dtype=np.float64)
    lse = np.empty((b, h, n), dtype=np.float64)
    for bi in range(b):
        for hi in range(h):
            o[bi, hi], lse[bi, hi] = forward_head(q[bi, hi], k[bi, hi], v[bi, hi], scale, causal)
    return o, lse


# ---------------------------------------------------------------------------
# Backward: standard attention backward
# ---------------------------------------------------------------------------

def softmax_backward_row(p: np.ndarray, dp: np.ndarray) -> np.ndarray:
    """ds = (diag(p) - p p^T) dp, written as the matrix product."""
    p = np.asarray(p, dtype=np.float64)
    dp = np.asarray(dp, dtype=np.float64)
    if p.shape != dp.shape or p.ndim != 1:
        raise ValueError("p and dp must be vectors of equal length")
    jac = np.diag(p) - np.outer(p, p)
    return jac @ dp


def backward_head(q, k, v, do, scale: float, causal: bool):
    """One head of the standard backward, with the softmax scale
    carried by dS (R1):

        dV = P^T dO
        dP = dO V^T
        dS = dsoftmax(dP), row-wise
           = P o (dP - D 1^T),  D_i = sum_j P_ij dP_ij   (Jacobian form)
        dQ = scale * dS K
        dK = scale * dS^T Q

    D is computed in the Jacobian form (rowsum(P o dP)), deliberately NOT as
    rowsum(dO o O), so that the identity between the two is a check.
    Returns (dQ, dK, dV, D) in float64.
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    s = scores(q, k, scale, causal)
    p, _, _ = softmax_rows(s)
    dv = p.T @ do
    dp = do @ v.T
    dd = np.sum(p * dp, axis=1)
    ds = p * (dp - dd[:, None])
    sc = as_f64_scale(scale)
    dq = sc * (ds @ k)
    dk = sc * (ds.T @ q)
    return dq, dk, dv, dd


def backward(q, k, v, do, scale: float, causal: bool):
    """Batched [B,H,N,d] backward.  Returns (dQ, dK, dV, D) float64."""
    q = np.asarray(q)
    b, h, n, d = q.shape
    dq = np.empty((b, h, n, d))
    dk = np.empty((b, h, n, d))
    dv = np.empty((b, h, n, d))
    dd = np.empty((b, h, n))
    for bi in range(b):
        for hi in range(h):
            dq[bi, hi], dk[bi, hi], dv[bi, hi], dd[bi, hi] = backward_head(
                q[bi, hi], k[bi, hi], v[bi, hi], do[bi, hi], scale, causal)
    return dq, dk, dv, dd


def rowsum_dO_O(o, do) -> np.ndarray:
    """D = rowsum(dO o O)  (Alg. 2 line 4; D has length N, R5).
    Works on [..., N, d] arrays; returns [..., N] float64."""
    o = np.asarray(o, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    return np.sum(do * o, axis=-1)


# ---------------------------------------------------------------------------
# Large-N variants: the same per-row definitions, evaluated row by row
# (O(N) memory per row instead of materialising N x N).  Each output row is
# computed by exactly the formulas above; rows are independent,
# so evaluating a chunk of rows at a time reorders nothing within a row.
# ---------------------------------------------------------------------------

def _row_chunks(n: int, rows_per_chunk: int):
    for r0 in range(0, n, rows_per_chunk):
        yield r0, min(n, r0 + rows_per_chunk)


def _row_scores(q_rows, row_idx, k, scale, causal):
    s = as_f64_scale(scale) * (q_rows @ k.T)
    if causal:
        cols = np.arange(k.shape[0])
        s[cols[None, :] > np.asarray(row_idx)[:, None]] = -np.inf
    return s


def forward_rows(q, k, v, scale: float, causal: bool, rows=None, rows_per_chunk: int = 256):
    """O and L for the given rows of one head (default: all rows), using the
    definitions of ``forward_head`` row by row.  Returns (rows, O[rows], L[rows])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n = q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows)
    o = np.empty((len(rows), v.shape[1]))
    lse = np.empty(len(rows))
    for a, b in _row_chunks(len(rows), rows_per_chunk):
        idx = rows[a:b]
        s = _row_scores(q[idx], idx, k, scale, causal)
        p, m, ell = softmax_rows(s)
        o[a:b] = p @ v
        lse[a:b] = m + np.log(ell)
    return rows, o, lse


def backward_sampled_head(q, k, v, do, scale: float, causal: bool, dq_rows, dkv_cols,
                          rows_per_chunk: int = 256):
    """Sampled backward for one head at large N (same definition as
    ``backward_head``):

      pass 1 (all rows i): L_i and D_i = sum_j P_ij dP_ij (Jacobian form);
      dQ_i = scale * sum_j P_ij (dP_ij - D_i) K_j          for i in dq_rows;
      dV_j = sum_i P_ij dO_i,  dK_j = scale * sum_i dS_ij Q_i   for j in dkv_cols.

    Returns dict with keys rows, dq, cols, dk, dv, lse (all rows), D (all rows).
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    n = q.shape[0]
    sc = as_f64_scale(scale)
    lse = np.empty(n)
    dd = np.empty(n)
    for a, b in _row_chunks(n, rows_per_chunk):
        idx = np.arange(a, b)
        s = _row_scores(q[a:b], idx, k, scale, causal)
        p, m, ell = softmax_rows(s)
        lse[a:b] = m + np.log(ell)
        dp = do[a:b] @ v.T
        dd[a:b] = np.sum(p * dp, axis=1)
    dq_rows = np.asarray(dq_rows)
    s = _row_scores(q[dq_rows], dq_rows, k, scale, causal)
    p = np.exp(s - lse[dq_rows][:, None])
    dp = do[dq_rows] @ v.T
    ds = p * (dp - dd[dq_rows][:, None])
    dq = sc * (ds @ k)
    # columns j: P_ij for all rows i, from L (P = exp(S - L), Alg. 2 line 11)
    dkv_cols = np.asarray(dkv_cols)
    st = sc * (k[dkv_cols] @ q.T)                      # [cols, N] = S^T for sampled cols
    if causal:
        st[np.arange(n)[None, :] < dkv_cols[:, None]] = -np.inf
    pt = np.exp(st - lse[None, :])
    dv = pt @ do
    dpt = v[dkv_cols] @ do.T
    dst = pt * (dpt - dd[None, :])
    dk = sc * (dst @ q)
    return {"rows": dq_rows, "dq": dq, "cols": dkv_cols, "dk": dk, "dv": dv,
            "lse": lse, "D": dd}


def naive_softmax_no_max(s: np.ndarray) -> np.ndarray:
    """softmax WITHOUT the max subtraction, used only by the overflow test
     to show why m is tracked."""
    with np.errstate(over="ignore", invalid="ignore"):
        e = np.exp(s)
        return e / np.sum(e, axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# MQA / GQA: query head h uses key/value head h // group, where
# group = H / H_kv; "implicitly manipulate the indices into the head" for the
# forward, and "sum the gradients dK and dV across different heads that were
# implicitly duplicated" for the backward.
# ---------------------------------------------------------------------------

def forward_gqa(q, k, v, scale: float, causal: bool):
    """q [B,H,N,d], k/v [B,H_kv,N,d] -> (O [B,H,N,d], L [B,H,N])."""
    q = np.asarray(q)
    b, h, n, d = q.shape
    h_kv = np.asarray(k).shape[1]
    if h % h_kv:
        raise ValueError("H must be a multiple of H_kv")
    group = h // h_kv
    o = np.empty((b, h, n, d))
    lse = np.empty((b, h, n))
    for bi in range(b):
        for hi in range(h):
            o[bi, hi], lse[bi, hi] = forward_head(q[bi, hi], k[bi, hi // group], v[bi, hi // group], scale, causal)
    return o, lse


def backward_gqa(q, k, v, do, scale: float, causal: bool):
    """Returns (dQ [B,H,N,d], dK [B,H_kv,N,d], dV [B,H_kv,N,d]); dK/dV of a
    key/value head are the sums over the query heads of its group."""
    q = np.asarray(q)
    b, h, n, d = q.shape
    h_kv = np.asarray(k).shape[1]
    group = h // h_kv
    dq = np.empty((b, h, n, d))
    dk = np.zeros((b, h_kv, n, d))
    dv = np.zeros((b, h_kv, n, d))
    for bi in range(b):
        for hi in range(h):
            g = hi // group
            dq[bi, hi], dkh, dvh, _ = backward_head(q[bi, hi], k[bi, g], v[bi, g], do[bi, hi], scale, causal)
            dk[bi, g] += dkh
            dv[bi, g] += dvh
    return dq, dk, dv


# ---------------------------------------------------------------------------
# N_q != N_k and variable-length batches.  The paper defines
# causal masking only for N_q == N_k; readings:
#   R22  causal with N_q != N_k is aligned to the BOTTOM-RIGHT corner: query
#        row i (0-based) sees key j iff j <= i + (N_k - N_q).  For N_q == N_k
#        this is exactly the mask of ``scores``.
#   R23  a query row that sees no key (possible when N_q > N_k, causal, or
#        N_k == 0) has O_i = 0 and L_i = -inf (the log of an empty sum); it
#        contributes nothing to any gradient.
# Variable-length batches use the packed layout: q [T_q, H, d], k and v
# [T_k, H_kv, d], sequence b = rows cu_q[b]:cu_q[b+1] of q and cu_k[b]:cu_k[b+1]
# of k/v; L is [H, T_q].  Every sequence is an independent attention problem
# (the per-(b,h) independence of P:162-165).
# ---------------------------------------------------------------------------

def scores_general(q, k, scale: float, causal: bool) -> np.ndarray:
    """S = scale * Q K^T [N_q, N_k]; causal mask bottom-right aligned (R22)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    s = as_f64_scale(scale) * (q @ k.T)
    if causal:
        n_q, n_k = s.shape
        rows = np.arange(n_q)[:, None]
        cols = np.arange(n_k)[None, :]
        s = np.where(cols > rows + (n_k - n_q), -np.inf, s)
    return s


def softmax_rows_general(s: np.ndarray):
    """``softmax_rows`` extended to rows with no finite entry (R23):
    for those m = -inf, l = 0 and the row of P is 0.  Returns (P, m, l)."""
    n_q = s.shape[0]
    m = np.max(s, axis=1) if s.shape[1] > 0 else np.full(n_q, -np.inf)
    finite = np.isfinite(m)
    e = np.exp(s - np.where(finite, m, 0.0)[:, None])       # exp(-inf) = 0 on empty rows
    ell = np.sum(e, axis=1)
    p = np.where(ell[:, None] > 0, e / np.where(ell > 0, ell, 1.0)[:, None], 0.0)
    return p, m, ell


def forward_head_general(q, k, v, scale: float, causal: bool):
    """One head, N_q x N_k (R22, R23): O = P V, L = m + log l (-inf on empty rows)."""
    v = np.asarray(v, dtype=np.float64)
    s = scores_general(q, k, scale, causal)
    p, m, ell = softmax_rows_general(s)
    o = p @ v if v.shape[0] > 0 else np.zeros((s.shape[0], v.shape[1]))
    with np.errstate(divide="ignore"):
        lse = np.where(ell > 0, m + np.log(np.where(ell > 0, ell, 1.0)), -np.inf)
    return o, lse


def backward_head_general(q, k, v, do, scale: float, causal: bool):
    """The backward of ``backward_head`` for N_q x N_k (R22, R23).
    Returns (dQ [N_q,d], dK [N_k,d], dV [N_k,d], D [N_q])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    s = scores_general(q, k, scale, causal)
    p, _, _ = softmax_rows_general(s)
    dv = p.T @ do
    dp = do @ v.T
    dd = np.sum(p * dp, axis=1)
    ds = p * (dp - dd[:, None])
    sc = as_f64_scale(scale)
    return sc * (ds @ k), sc * (ds.T @ q), dv, dd


def _check_cu(cu, total, name):
    cu = np.asarray(cu, dtype=np.int64)
    if cu.ndim != 1 or len(cu) < 2 or cu[0] != 0 or cu[-1] != total or np.any(np.diff(cu) < 0):
        raise ValueError(f"{name} must be non-decreasing, start at 0 and end at {total}")
    return cu


def forward_varlen(q, k, v, cu_q, cu_k, scale: float, causal: bool):
    """Packed variable-length batch: q [T_q,H,d], k/v [T_k,H_kv,d] ->
    (O [T_q,H,d], L [H,T_q]).  Query head h uses key/value head h // (H/H_kv)
    (P:444-452)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    t_q, h, d = q.shape
    h_kv = k.shape[1]
    group = h // h_kv
    cu_q = _check_cu(cu_q, t_q, "cu_q")
    cu_k = _check_cu(cu_k, k.shape[0], "cu_k")
    o = np.zeros((t_q, h, v.shape[2]))
    lse = np.full((h, t_q), -np.inf)
    for b in range(len(cu_q) - 1):
        qs, qe, ks, ke = cu_q[b], cu_q[b + 1], cu_k[b], cu_k[b + 1]
        for hi in range(h):
            o[qs:qe, hi], lse[hi, qs:qe] = forward_head_general(
                q[qs:qe, hi], k[ks:ke, hi // group], v[ks:ke, hi // group], scale, causal)
    return o, lse


def backward_varlen(q, k, v, do, cu_q, cu_k, scale: float, causal: bool):
    """Packed variable-length backward: returns (dQ [T_q,H,d], dK [T_k,H_kv,d],
    dV [T_k,H_kv,d]); dK/dV of a key/value head sum over its query heads."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    t_q, h, d = q.shape
    h_kv = k.shape[1]
    group = h // h_kv
    cu_q = _check_cu(cu_q, t_q, "cu_q")
    cu_k = _check_cu(cu_k, k.shape[0], "cu_k")
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for b in range(len(cu_q) - 1):
        qs, qe, ks, ke = cu_q[b], cu_q[b + 1], cu_k[b], cu_k[b + 1]
        for hi in range(h):
            g = hi // group
            gq, gk, gv, _ = backward_head_general(q[qs:qe, hi], k[ks:ke, g], v[ks:ke, g], do[qs:qe, hi],
                                                  scale, causal)
            dq[qs:qe, hi] = gq
            dk[ks:ke, g] += gk
            dv[ks:ke, g] += gv
    return dq, dk, dv


# ---------------------------------------------------------------------------
# FP8 forward (the paper names FP8 as future work).
# The inputs are E4M3 numbers x8 with fp32 descales: the represented values
# descale_x * x8 are exact in float64, so the expected O and L are the plain
# definition (``forward_gqa``) on them.  The kernel's own rounding of P~ to E4M3
# (R25) is a kernel contract; its tolerance model lives with the tests
# (tests/fp8_bound.py), not here.
# ---------------------------------------------------------------------------
