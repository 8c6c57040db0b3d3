"""Pins for the CPU fp64 oracle (oracle/ref_attention.py, oracle/flops.py).

Each test checks the oracle against something other than itself: values the
paper/spec print (tests/golden/worked_examples.json, cited there), closed
forms, invariants that the mathematics fixes, brute-force pure-Python loops,
and central finite differences.  Chosen so that a dropped term, a wrong sign
or index, a transposed operand or a missing scale fails at least one test.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import flops as F
from oracle import ref_attention as R
from tests.fp8_bound import fp8_pv_error_bound

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def rng(seed):
    return np.random.default_rng(seed)


# --------------------------------------------------------------------------
# Worked values printed in SPEC.md / PAPER.md
# --------------------------------------------------------------------------

def test_golden_two_step_online_softmax():
    g = GOLD["two_step_online_softmax"]
    # one query row whose scores against the two keys are S_row = [0, 0]
    q = np.array([[0.0]])
    k = np.array([[0.0], [0.0]])
    o, lse = R.forward_head(q, k, np.array(g["V"]), scale=1.0, causal=False)
    assert np.allclose(o, g["O"], atol=1e-15)
    assert np.allclose(lse, g["L"], atol=1e-15)


def test_golden_finalize_output():
    g = GOLD["finalize_output"]
    # scores [1, 1] give m = 1, l = 2; V rows sum to O_accum = [4, 6]
    q = np.array([[1.0]])
    k = np.array([[1.0], [1.0]])
    v = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.allclose(v.sum(0), g["O_accum"])
    p, m, ell = R.softmax_rows(R.scores(q, k, 1.0, False))
    assert m[0] == g["m"] and abs(ell[0] - g["ell"]) < 1e-15
    o, lse = R.forward_head(q, k, v, 1.0, False)
    assert np.allclose(o[0], g["O"], atol=1e-15)
    assert abs(lse[0] - g["L"]) < 1e-12


def test_golden_softmax_backward_row():
    g = GOLD["softmax_backward_row"]
    ds = R.softmax_backward_row(np.array(g["p"]), np.array(g["dp"]))
    assert np.allclose(ds, g["ds"], atol=1e-15)
    # constant dp -> ds = 0
    p = rng(1).dirichlet(np.ones(16))
    assert np.allclose(R.softmax_backward_row(p, np.full(16, 3.7)), 0.0, atol=1e-14)


def test_golden_compute_D():
    g = GOLD["compute_D"]
    d = R.rowsum_dO_O(np.array([g["O"]]), np.array([g["dO"]]))
    assert d[0] == g["D"]


def test_golden_rowmax_rowsum():
    g = GOLD["rowmax_rowsum"]
    _, m, _ = R.softmax_rows(np.array(g["rowmax_in"]))
    assert list(m) == g["rowmax_out"]
    # ell of S - m + log(x) recovers rowsum(x) for positive x: exp(log x) summed
    x = np.array(g["rowsum_in"])
    _, m2, ell = R.softmax_rows(np.log(x))
    assert np.allclose(ell * np.exp(m2), g["rowsum_out"], atol=1e-12)


def test_golden_flops():
    g = GOLD["flops"]
    assert F.attention_flops(g["batch"], g["heads"], g["N"], g["d"], False) == g["fwd"]
    assert F.attention_flops(g["batch"], g["heads"], g["N"], g["d"], True) == g["fwd_causal"]
    assert F.attention_flops(g["batch"], g["heads"], g["N"], g["d"], False, "bwd") == g["bwd"]
    assert F.attention_flops(2, g["heads"], g["N"], g["d"], False) == 2 * g["fwd"]


def test_golden_causal_census():
    g = GOLD["causal_census"]
    c = F.causal_census(g["N"], g["Br"], g["Bc"])
    assert (c["full"], c["partial"], c["skip"]) == (g["full"], g["partial"], g["skip"])


@pytest.mark.parametrize("t", [1, 2, 3, 5, 8])
def test_census_square_closed_form(t):
    # square tiling with T tiles: T(T+1)/2 computed, T partial, T(T-1)/2 skipped
    c = F.causal_census(16 * t, 16, 16)
    assert c["partial"] == t
    assert c["full"] + c["partial"] == t * (t + 1) // 2
    assert c["skip"] == t * (t - 1) // 2


def test_census_ragged_and_rectangular():
    # Br != Bc: more than one partial block per row block can occur (R8)
    c = F.causal_census(100, 32, 16)
    for i, cols in enumerate(c["computed"]):
        last_row = min(100, (i + 1) * 32) - 1
        assert cols == list(range(last_row // 16 + 1))


# --------------------------------------------------------------------------
# Brute force: pure-Python loops on tiny inputs (independent of numpy matmul)
# --------------------------------------------------------------------------

def _brute_forward(q, k, v, scale, causal):
    n, d = len(q), len(q[0])
    o, lse = [], []
    for i in range(n):
        s = []
        for j in range(len(k)):
            if causal and j > i:
                continue
            s.append((j, scale * math.fsum(q[i][t] * k[j][t] for t in range(d))))
        mx = max(x for _, x in s)
        den = math.fsum(math.exp(x - mx) for _, x in s)
        row = [math.fsum(math.exp(x - mx) / den * v[j][c] for j, x in s) for c in range(len(v[0]))]
        o.append(row)
        lse.append(mx + math.log(den))
    return np.array(o), np.array(lse)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("n,d", [(1, 3), (5, 4), (9, 2)])
def test_forward_matches_brute_force(n, d, causal):
    r = rng(n * 10 + d)
    q, k, v = r.normal(size=(3, n, d))
    scale = float(np.float32(1 / math.sqrt(d)))
    o, lse = R.forward_head(q, k, v, scale, causal)
    ob, lb = _brute_forward(q.tolist(), k.tolist(), v.tolist(), scale, causal)
    assert np.max(np.abs(o - ob)) < 1e-13
    assert np.max(np.abs(lse - lb)) < 1e-13


def _brute_backward(q, k, v, do, scale, causal):
    """dQ, dK, dV by the element-wise chain rule written as loops."""
    n, d = q.shape
    s = np.full((n, n), -np.inf)
    for i in range(n):
        for j in range(n):
            if not (causal and j > i):
                s[i, j] = scale * sum(q[i, t] * k[j, t] for t in range(d))
    p = np.zeros((n, n))
    for i in range(n):
        mx = max(s[i])
        den = sum(math.exp(x - mx) for x in s[i] if x != -np.inf)
        for j in range(n):
            p[i, j] = 0.0 if s[i, j] == -np.inf else math.exp(s[i, j] - mx) / den
    dq = np.zeros((n, d)); dk = np.zeros((n, d)); dv = np.zeros((n, d))
    for i in range(n):
        dp = [sum(do[i, t] * v[j, t] for t in range(d)) for j in range(n)]
        for j in range(n):
            ds = sum(p[i, j] * ((1.0 if a == j else 0.0) - p[i, a]) * dp[a] for a in range(n))
            for t in range(d):
                dq[i, t] += scale * ds * k[j, t]
                dk[j, t] += scale * ds * q[i, t]
                dv[j, t] += p[i, j] * do[i, t]
    return dq, dk, dv


@pytest.mark.parametrize("causal", [False, True])
def test_backward_matches_brute_force(causal):
    r = rng(7)
    q, k, v, do = r.normal(size=(4, 6, 3))
    scale = 0.7
    dq, dk, dv, _ = R.backward_head(q, k, v, do, scale, causal)
    bq, bk, bv = _brute_backward(q, k, v, do, float(np.float32(scale)), causal)
    for a, b in ((dq, bq), (dk, bk), (dv, bv)):
        assert np.max(np.abs(a - b)) < 1e-13


# --------------------------------------------------------------------------
# Closed forms
# --------------------------------------------------------------------------

@pytest.mark.parametrize("causal", [False, True])
def test_identical_keys_closed_form(causal):
    r = rng(3)
    n, d = 40, 8
    q = r.normal(size=(n, d))
    krow = r.normal(size=d)
    k = np.tile(krow, (n, 1))
    v = r.normal(size=(n, d))
    do = r.normal(size=(n, d))
    s = 0.35
    sc = float(np.float32(s))
    o, lse = R.forward_head(q, k, v, s, causal)
    if causal:
        want = np.cumsum(v, axis=0) / np.arange(1, n + 1)[:, None]
        want_l = sc * (q @ krow) + np.log(np.arange(1, n + 1))
    else:
        want = np.tile(v.mean(0), (n, 1))
        want_l = sc * (q @ krow) + np.log(n)
    assert np.max(np.abs(o - want)) < 1e-13
    assert np.max(np.abs(lse - want_l)) < 1e-13
    dq, dk, dv, _ = R.backward_head(q, k, v, do, s, causal)
    assert np.max(np.abs(dq)) < 1e-13  # logits of a row are all equal for every q


@pytest.mark.parametrize("causal", [False, True])
def test_one_hot_large_logit(causal):
    n, d, jstar, alpha = 64, 64, 17, 32.0
    q = np.zeros((n, d)); q[:, 0] = alpha
    k = np.zeros((n, d)); k[jstar, 0] = alpha
    v = rng(5).normal(size=(n, d))
    s = 1 / math.sqrt(d)        # s * alpha^2 = 128
    o, _ = R.forward_head(q, k, v, s, causal)
    rows = np.arange(jstar, n) if causal else np.arange(n)
    assert np.max(np.abs(o[rows] - v[jstar])) < n * math.exp(-120)
    if causal:  # rows before j* see only zero logits: uniform prefix mean
        for i in range(jstar):
            assert np.allclose(o[i], v[: i + 1].mean(0), atol=1e-13)


def test_causal_row0_and_N1():
    r = rng(11)
    q, k, v, do = r.normal(size=(4, 9, 5))
    o, lse = R.forward_head(q, k, v, 0.5, True)
    assert np.array_equal(o[0], v[0])
    assert abs(lse[0] - 0.5 * q[0] @ k[0]) < 1e-15
    o1, l1 = R.forward_head(q[:1], k[:1], v[:1], 0.5, False)
    assert np.array_equal(o1, v[:1])
    dq, dk, dv, _ = R.backward_head(q[:1], k[:1], v[:1], do[:1], 0.5, False)
    assert np.array_equal(dv, do[:1])
    assert np.all(dq == 0) and np.all(dk == 0)


def test_zero_query_uniform():
    r = rng(12)
    k, v = r.normal(size=(2, 4, 2))
    p, _, _ = R.softmax_rows(R.scores(np.zeros((4, 2)), k, 1.0, False))
    assert np.allclose(p, 0.25, atol=1e-16)
    o, _ = R.forward_head(np.zeros((4, 2)), k, v, 1.0, False)
    assert np.allclose(o, v.mean(0), atol=1e-15)


def test_dO_zero_gives_zero_grads():
    r = rng(13)
    q, k, v = r.normal(size=(3, 10, 4))
    for causal in (False, True):
        dq, dk, dv, dd = R.backward_head(q, k, v, np.zeros((10, 4)), 0.5, causal)
        assert not dq.any() and not dk.any() and not dv.any() and not dd.any()


# --------------------------------------------------------------------------
# Invariants
# --------------------------------------------------------------------------

@pytest.mark.parametrize("causal", [False, True])
def test_rows_sum_to_one_and_mask(causal):
    r = rng(21)
    q, k = r.normal(size=(2, 33, 8))
    p, _, _ = R.softmax_rows(R.scores(q, k, 0.3, causal))
    assert np.max(np.abs(p.sum(1) - 1)) < 1e-14
    assert np.all(p >= 0) and np.all(p <= 1)
    if causal:
        assert np.all(p[np.triu_indices(33, 1)] == 0)


def test_shift_invariance():
    r = rng(22)
    s = r.normal(size=(7, 11)) * 4
    p0, _, _ = R.softmax_rows(s)
    p1, _, _ = R.softmax_rows(s + r.normal(size=(7, 1)) * 50)
    assert np.max(np.abs(p0 - p1)) < 1e-14


def test_logsumexp_identity():
    r = rng(23)
    q, k = r.normal(size=(2, 12, 4))
    for causal in (False, True):
        _, lse = R.forward_head(q, k, np.eye(12, 4), 0.8, causal)
        sc = float(np.float32(0.8))
        for i in range(12):
            js = range(i + 1) if causal else range(12)
            tot = math.fsum(math.exp(sc * float(q[i] @ k[j])) for j in js)
            assert abs(math.exp(lse[i]) - tot) < 1e-12 * tot


def test_two_block_identity():
    """P:328-335 (with the rescale factor e^{m1-m2}, no inverse, R3): the
    statistics after two blocks equal rowmax / rowsum over the full row."""
    r = rng(24)
    s = r.normal(size=(5, 32)) * 3
    _, m, ell = R.softmax_rows(s)
    s1, s2 = s[:, :16], s[:, 16:]
    m1 = s1.max(1); l1 = np.exp(s1 - m1[:, None]).sum(1)
    m2 = np.maximum(m1, s2.max(1))
    l2 = np.exp(m1 - m2) * l1 + np.exp(s2 - m2[:, None]).sum(1)
    assert np.array_equal(m2, m) and np.max(np.abs(l2 - ell)) < 1e-13


def test_key_permutation_invariance():
    r = rng(25)
    q, k, v = r.normal(size=(3, 20, 6))
    perm = r.permutation(20)
    o0, l0 = R.forward_head(q, k, v, 0.4, False)
    o1, l1 = R.forward_head(q, k[perm], v[perm], 0.4, False)
    assert np.max(np.abs(o0 - o1)) < 1e-14 and np.max(np.abs(l0 - l1)) < 1e-14


def test_causal_perturbation_locality():
    r = rng(26)
    q, k, v = r.normal(size=(3, 128, 8))
    o0, _ = R.forward_head(q, k, v, 0.3, True)
    k2 = k.copy(); k2[100] += 5.0
    v2 = v.copy(); v2[100] -= 3.0
    o1, _ = R.forward_head(q, k2, v2, 0.3, True)
    assert np.array_equal(o0[:100], o1[:100])
    assert not np.allclose(o0[100:], o1[100:])


def test_overflow_robustness():
    r = rng(27)
    # S:234 uses +300, which overflows exp in fp32 (the kernel's type); fp64
    # exp overflows above ~709, so the oracle is pinned at logits up to +800.
    s = r.uniform(700, 800, size=(4, 9))
    p, m, ell = R.softmax_rows(s)
    assert np.all(np.isfinite(p)) and np.all(np.isfinite(m + np.log(ell)))
    assert not np.all(np.isfinite(R.naive_softmax_no_max(s)))


@pytest.mark.parametrize("causal", [False, True])
def test_D_identity_and_gradient_sums(causal):
    r = rng(28)
    q, k, v, do = r.normal(size=(4, 30, 8))
    o, _ = R.forward_head(q, k, v, 0.4, causal)
    dq, dk, dv, dd = R.backward_head(q, k, v, do, 0.4, causal)
    # D (Jacobian form) == rowsum(dO o O)
    assert np.max(np.abs(dd - R.rowsum_dO_O(o, do))) < 1e-12
    # sum_j dK_j = 0: softmax is invariant to a common shift of every key
    assert np.max(np.abs(dk.sum(0))) < 1e-12
    # sum_j dV_j = sum_i dO_i: rows of P sum to 1
    assert np.max(np.abs(dv.sum(0) - do.sum(0))) < 1e-12


# --------------------------------------------------------------------------
# Finite differences
# --------------------------------------------------------------------------

@pytest.mark.parametrize("causal", [False, True])
def test_finite_differences(causal):
    r = rng(31)
    n, d = 13, 5
    q, k, v, g = r.normal(size=(4, n, d))
    scale = float(np.float32(0.6))
    dq, dk, dv, _ = R.backward_head(q, k, v, g, scale, causal)
    h = 1e-6

    def f(qq, kk, vv):
        o, _ = R.forward_head(qq, kk, vv, scale, causal)
        return float(np.sum(o * g))

    for which, grad in ((0, dq), (1, dk), (2, dv)):
        for (i, t) in [(0, 0), (3, 2), (n - 1, d - 1), (7, 1)]:
            args = [q.copy(), k.copy(), v.copy()]
            args[which][i, t] += h
            fp = f(*args)
            args[which][i, t] -= 2 * h
            fm = f(*args)
            fd = (fp - fm) / (2 * h)
            assert abs(fd - grad[i, t]) < 1e-7, (which, i, t, fd, grad[i, t])


def test_finite_difference_softmax_row():
    r = rng(32)
    s = r.normal(size=16)
    dp = r.normal(size=16)
    p, _, _ = R.softmax_rows(s[None])
    ds = R.softmax_backward_row(p[0], dp)
    h = 1e-6
    for j in range(16):
        e = np.zeros(16); e[j] = h
        fp = R.softmax_rows((s + e)[None])[0][0] @ dp
        fm = R.softmax_rows((s - e)[None])[0][0] @ dp
        assert abs((fp - fm) / (2 * h) - ds[j]) < 1e-8


# --------------------------------------------------------------------------
# Large-N (row-streamed) variants agree with the materialising definition
# --------------------------------------------------------------------------

@pytest.mark.parametrize("causal", [False, True])
def test_sampled_variants_match_full(causal):
    r = rng(41)
    n, d = 300, 16
    q, k, v, do = r.normal(size=(4, n, d))
    o, lse = R.forward_head(q, k, v, 0.25, causal)
    rows, o2, l2 = R.forward_rows(q, k, v, 0.25, causal, rows=[0, 5, 128, 299], rows_per_chunk=3)
    assert np.max(np.abs(o2 - o[rows])) < 1e-13 and np.max(np.abs(l2 - lse[rows])) < 1e-13
    dq, dk, dv, dd = R.backward_head(q, k, v, do, 0.25, causal)
    sm = R.backward_sampled_head(q, k, v, do, 0.25, causal, dq_rows=[0, 77, 299],
                                 dkv_cols=[0, 150, 299], rows_per_chunk=64)
    assert np.max(np.abs(sm["dq"] - dq[sm["rows"]])) < 1e-12
    assert np.max(np.abs(sm["dk"] - dk[sm["cols"]])) < 1e-12
    assert np.max(np.abs(sm["dv"] - dv[sm["cols"]])) < 1e-12
    assert np.max(np.abs(sm["D"] - dd)) < 1e-12 and np.max(np.abs(sm["lse"] - lse)) < 1e-12


def test_batched_wrappers():
    r = rng(42)
    q, k, v, do = r.normal(size=(4, 2, 3, 10, 4))
    o, lse = R.forward(q, k, v, 0.5, True)
    dq, dk, dv, dd = R.backward(q, k, v, do, 0.5, True)
    for b in range(2):
        for h in range(3):
            o1, l1 = R.forward_head(q[b, h], k[b, h], v[b, h], 0.5, True)
            assert np.array_equal(o[b, h], o1) and np.array_equal(lse[b, h], l1)
            g = R.backward_head(q[b, h], k[b, h], v[b, h], do[b, h], 0.5, True)
            assert np.array_equal(dq[b, h], g[0]) and np.array_equal(dv[b, h], g[2])


# --------------------------------------------------------------------------
# MQA / GQA
# --------------------------------------------------------------------------

@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("h,h_kv", [(4, 4), (4, 2), (6, 1)])
def test_gqa_equals_explicit_duplication(h, h_kv, causal):
    """GQA through index manipulation == MHA on explicitly repeated K/V, with
    dK/dV of the duplicated heads summed back (the paper's two statements)."""
    r = rng(50 + h + h_kv)
    b, n, d = 2, 11, 4
    q = r.normal(size=(b, h, n, d))
    k = r.normal(size=(b, h_kv, n, d))
    v = r.normal(size=(b, h_kv, n, d))
    do = r.normal(size=(b, h, n, d))
    grp = h // h_kv
    kr, vr = np.repeat(k, grp, axis=1), np.repeat(v, grp, axis=1)
    o, lse = R.forward_gqa(q, k, v, 0.5, causal)
    o2, l2 = R.forward(q, kr, vr, 0.5, causal)
    assert np.array_equal(o, o2) and np.array_equal(lse, l2)
    dq, dk, dv = R.backward_gqa(q, k, v, do, 0.5, causal)
    dq2, dk2, dv2, _ = R.backward(q, kr, vr, do, 0.5, causal)
    assert np.max(np.abs(dq - dq2)) < 1e-13
    assert np.max(np.abs(dk - dk2.reshape(b, h_kv, grp, n, d).sum(2))) < 1e-12
    assert np.max(np.abs(dv - dv2.reshape(b, h_kv, grp, n, d).sum(2))) < 1e-12


def test_gqa_finite_differences():
    r = rng(61)
    b, h, h_kv, n, d = 1, 4, 2, 7, 3
    q = r.normal(size=(b, h, n, d))
    k = r.normal(size=(b, h_kv, n, d))
    v = r.normal(size=(b, h_kv, n, d))
    g = r.normal(size=(b, h, n, d))
    dq, dk, dv = R.backward_gqa(q, k, v, g, 0.7, True)
    f = lambda qq, kk, vv: float(np.sum(R.forward_gqa(qq, kk, vv, 0.7, True)[0] * g))
    eps = 1e-6
    for which, grad, idx in ((1, dk, (0, 1, 3, 2)), (2, dv, (0, 0, 5, 1)), (0, dq, (0, 3, 6, 0))):
        args = [q.copy(), k.copy(), v.copy()]
        args[which][idx] += eps
        fp = f(*args)
        args[which][idx] -= 2 * eps
        fm = f(*args)
        assert abs((fp - fm) / (2 * eps) - grad[idx]) < 1e-7


# --------------------------------------------------------------------------
# N_q != N_k (bottom-right causal, R22), empty rows (R23), packed varlen
# --------------------------------------------------------------------------

def _brute_general(q, k, v, do, scale, causal):
    """Pure-Python loops: forward O, L and backward dQ, dK, dV for an N_q x N_k
    head with the bottom-right causal mask (j visible iff j <= i + N_k - N_q);
    rows with no visible key give O = 0, L = -inf and no gradient."""
    nq, nk, d = len(q), len(k), len(q[0])
    off = nk - nq
    o = [[0.0] * len(v[0]) if nk else [0.0] * d for _ in range(nq)]
    lse = [-math.inf] * nq
    p = [[0.0] * nk for _ in range(nq)]
    for i in range(nq):
        vis = [j for j in range(nk) if not (causal and j > i + off)]
        if not vis:
            continue
        s = {j: scale * math.fsum(q[i][t] * k[j][t] for t in range(d)) for j in vis}
        mx = max(s.values())
        den = math.fsum(math.exp(x - mx) for x in s.values())
        for j in vis:
            p[i][j] = math.exp(s[j] - mx) / den
        o[i] = [math.fsum(p[i][j] * v[j][c] for j in vis) for c in range(len(v[0]))]
        lse[i] = mx + math.log(den)
    dq = [[0.0] * d for _ in range(nq)]
    dk = [[0.0] * d for _ in range(nk)]
    dv = [[0.0] * len(v[0]) for _ in range(nk)]
    for i in range(nq):
        dp = [math.fsum(do[i][t] * v[j][t] for t in range(len(v[0]))) for j in range(nk)]
        for j in range(nk):
            ds = math.fsum(p[i][j] * ((1.0 if a == j else 0.0) - p[i][a]) * dp[a] for a in range(nk))
            for t in range(d):
                dq[i][t] += scale * ds * k[j][t]
                dk[j][t] += scale * ds * q[i][t]
            for t in range(len(v[0])):
                dv[j][t] += p[i][j] * do[i][t]
    return [np.array(x, dtype=np.float64) for x in (o, lse, dq, dk, dv)]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("nq,nk", [(3, 7), (7, 3), (5, 5), (1, 4), (4, 1), (6, 0)])
def test_general_matches_brute_force(nq, nk, causal):
    r = rng(100 + 10 * nq + nk)
    d = 3
    q, do = r.normal(size=(2, nq, d))
    k, v = r.normal(size=(2, nk, d))
    scale = float(np.float32(0.8))
    o, lse = R.forward_head_general(q, k, v, scale, causal)
    dq, dk, dv, _ = R.backward_head_general(q, k, v, do, scale, causal)
    bo, bl, bq, bk, bv = _brute_general(q.tolist(), k.tolist(), v.tolist(), do.tolist(), scale, causal)
    assert np.max(np.abs(o - bo), initial=0) < 1e-13
    assert np.array_equal(np.isinf(lse), np.isinf(bl))
    fin = np.isfinite(bl)
    assert np.max(np.abs(lse[fin] - bl[fin]), initial=0) < 1e-13
    for a, b in ((dq, bq), (dk, bk), (dv, bv)):
        assert np.max(np.abs(a - np.reshape(b, a.shape)), initial=0) < 1e-12


@pytest.mark.parametrize("causal", [False, True])
def test_general_reduces_to_square(causal):
    """N_q == N_k: the bottom-right mask is the paper's mask."""
    r = rng(120)
    q, k, v, do = r.normal(size=(4, 9, 4))
    o, lse = R.forward_head_general(q, k, v, 0.5, causal)
    o2, l2 = R.forward_head(q, k, v, 0.5, causal)
    assert np.max(np.abs(o - o2)) < 1e-15 and np.max(np.abs(lse - l2)) < 1e-15
    g = R.backward_head_general(q, k, v, do, 0.5, causal)
    g2 = R.backward_head(q, k, v, do, 0.5, causal)
    for a, b in zip(g, g2):
        assert np.max(np.abs(a - b)) < 1e-15


def test_general_closed_forms():
    r = rng(121)
    d = 4
    # N_q > N_k causal: the first N_q - N_k rows see nothing, row N_q - N_k sees key 0 only
    nq, nk = 9, 4
    q = r.normal(size=(nq, d)); k = r.normal(size=(nk, d)); v = r.normal(size=(nk, d))
    sc = float(np.float32(0.5))
    o, lse = R.forward_head_general(q, k, v, sc, True)
    assert np.all(o[:nq - nk] == 0) and np.all(lse[:nq - nk] == -np.inf)
    assert np.max(np.abs(o[nq - nk] - v[0])) < 1e-15
    assert abs(lse[nq - nk] - sc * float(q[nq - nk] @ k[0])) < 1e-14
    # N_q < N_k causal: row i is plain attention over the first i + N_k - N_q + 1 keys
    nq, nk = 4, 11
    q = r.normal(size=(nq, d)); k = r.normal(size=(nk, d)); v = r.normal(size=(nk, d))
    o, lse = R.forward_head_general(q, k, v, sc, True)
    for i in range(nq):
        m = i + nk - nq + 1
        oi, li = R.forward_head(q[i:i + 1], k[:m], v[:m], sc, False)
        assert np.max(np.abs(o[i] - oi[0])) < 1e-14 and abs(lse[i] - li[0]) < 1e-14
    # empty rows carry no gradient
    dq, dk, dv, dd = R.backward_head_general(q[:1].repeat(3, 0), k[:1], v[:1], r.normal(size=(3, d)), sc, True)
    assert np.all(dq[:2] == 0) and np.all(dd[:2] == 0)


@pytest.mark.parametrize("nq,nk", [(5, 8), (8, 5)])
def test_general_finite_differences(nq, nk):
    r = rng(122 + nq)
    d = 3
    q, g = r.normal(size=(2, nq, d))
    k, v = r.normal(size=(2, nk, d))
    sc = float(np.float32(0.6))
    dq, dk, dv, _ = R.backward_head_general(q, k, v, g, sc, True)

    def f(qq, kk, vv):
        return float(np.sum(R.forward_head_general(qq, kk, vv, sc, True)[0] * g))

    h = 1e-6
    for which, grad, idx in ((0, dq, (nq - 1, 1)), (0, dq, (nq // 2, 0)), (1, dk, (0, 2)), (1, dk, (nk - 1, 0)),
                             (2, dv, (1, 1)), (2, dv, (nk - 1, 2))):
        args = [q.copy(), k.copy(), v.copy()]
        args[which][idx] += h
        fp = f(*args)
        args[which][idx] -= 2 * h
        fm = f(*args)
        assert abs((fp - fm) / (2 * h) - grad[idx]) < 1e-7, (which, idx)


@pytest.mark.parametrize("causal", [False, True])
def test_varlen_matches_brute_force(causal):
    """Packed batch with an empty query sequence, N_q > N_k and N_q < N_k
    sequences, and GQA (H = 4 query heads on H_kv = 2)."""
    r = rng(130)
    cu_q = [0, 3, 3, 8, 10]
    cu_k = [0, 5, 7, 9, 9 + 6]
    h, h_kv, d = 4, 2, 3
    q = r.normal(size=(cu_q[-1], h, d)); do = r.normal(size=(cu_q[-1], h, d))
    k = r.normal(size=(cu_k[-1], h_kv, d)); v = r.normal(size=(cu_k[-1], h_kv, d))
    sc = float(np.float32(0.7))
    o, lse = R.forward_varlen(q, k, v, cu_q, cu_k, sc, causal)
    dq, dk, dv = R.backward_varlen(q, k, v, do, cu_q, cu_k, sc, causal)
    dk_b = np.zeros_like(k); dv_b = np.zeros_like(v)
    for b in range(len(cu_q) - 1):
        qs, qe, ks, ke = cu_q[b], cu_q[b + 1], cu_k[b], cu_k[b + 1]
        if qe == qs:   # an empty query sequence: nothing to compute, no gradient for its keys
            assert np.all(dk[ks:ke] == 0) and np.all(dv[ks:ke] == 0)
            continue
        for hi in range(h):
            g = hi // (h // h_kv)
            bo, bl, bq, bk, bv = _brute_general(q[qs:qe, hi].tolist(), k[ks:ke, g].tolist(), v[ks:ke, g].tolist(),
                                                do[qs:qe, hi].tolist(), sc, causal)
            if qe > qs:
                assert np.max(np.abs(o[qs:qe, hi] - bo)) < 1e-13
                fin = np.isfinite(bl)
                assert np.array_equal(np.isinf(lse[hi, qs:qe]), ~fin)
                assert np.max(np.abs(lse[hi, qs:qe][fin] - bl[fin]), initial=0) < 1e-13
                assert np.max(np.abs(dq[qs:qe, hi] - bq)) < 1e-12
            if ke > ks:
                dk_b[ks:ke, g] += bk
                dv_b[ks:ke, g] += bv
    assert np.max(np.abs(dk - dk_b)) < 1e-12 and np.max(np.abs(dv - dv_b)) < 1e-12


def test_varlen_finite_differences():
    r = rng(131)
    cu_q, cu_k = [0, 4, 9], [0, 6, 9]
    q = r.normal(size=(9, 2, 3)); g = r.normal(size=(9, 2, 3))
    k = r.normal(size=(9, 1, 3)); v = r.normal(size=(9, 1, 3))
    dq, dk, dv = R.backward_varlen(q, k, v, g, cu_q, cu_k, 0.9, True)
    f = lambda qq, kk, vv: float(np.sum(R.forward_varlen(qq, kk, vv, cu_q, cu_k, 0.9, True)[0] * g))
    h = 1e-6
    for which, grad, idx in ((0, dq, (8, 1, 2)), (1, dk, (7, 0, 1)), (2, dv, (2, 0, 0)), (1, dk, (0, 0, 2))):
        args = [q.copy(), k.copy(), v.copy()]
        args[which][idx] += h
        fp = f(*args)
        args[which][idx] -= 2 * h
        fm = f(*args)
        assert abs((fp - fm) / (2 * h) - grad[idx]) < 1e-7, (which, idx)


def test_varlen_rejects_bad_offsets():
    z = np.zeros((4, 1, 2))
    for cu in ([0, 5], [1, 4], [0, 3, 2, 4], [0]):
        with pytest.raises(ValueError):
            R.forward_varlen(z, z, z, cu, [0, 4], 1.0, False)


# --------------------------------------------------------------------------
# FP8 (R25): the P~V rounding bound
# --------------------------------------------------------------------------

def _e4m3_round(x):
    """Independent E4M3 round-to-nearest-even of non-negative values (max 448;
    normals 2^-6..448 with 3 mantissa bits, subnormals in steps of 2^-9)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = x > 0
    e = np.floor(np.log2(np.where(nz, x, 1.0)))
    e = np.maximum(e, -6)                      # below 2^-6: subnormal spacing 2^-9
    step = 2.0 ** (e - 3)
    out[nz] = (np.round(x[nz] / step[nz]) * step[nz])   # np.round: half to even
    return np.minimum(out, 448.0)


@pytest.mark.parametrize("causal", [False, True])
def test_fp8_bound_matches_brute_force_and_holds(causal):
    r = rng(140)
    n, d = 11, 4
    q, k, v = r.normal(size=(3, n, d))
    sc = 0.9
    bound = fp8_pv_error_bound(q, k, v, sc, causal)
    # brute force of the formula
    for i in range(n):
        vis = [j for j in range(n) if not (causal and j > i)]
        s = [float(np.float32(sc)) * float(q[i] @ k[j]) for j in vis]
        mx = max(s)
        e = [math.exp(x - mx) for x in s]
        l = math.fsum(e)
        for c in range(d):
            want = 2 ** -4 * math.fsum(e[t] / l * abs(v[j, c]) for t, j in enumerate(vis)) + \
                2 ** -10 / l * math.fsum(abs(v[j, c]) for j in vis)
            assert abs(bound[i, c] - want) < 1e-14
    # the bound holds for P~ rounded to E4M3 relative to any running max within 8 (log2) of the true max
    o, _ = R.forward_head(q, k, v, sc, causal)
    s_ = R.scores(q, k, sc, causal)
    for shift in (0.0, 3.0, 8.0):   # running max below the true max by `shift` (log2 units)
        m = np.max(s_, axis=1) - shift * math.log(2)
        pt = np.exp(s_ - m[:, None])
        o8 = (_e4m3_round(pt) @ v) / np.sum(pt, axis=1)[:, None]
        assert np.all(np.abs(o8 - o) <= bound + 1e-12)


def test_e4m3_rounding_helper():
    """The test's E4M3 rounding against torch's float8_e4m3fn cast."""
    import torch
    x = np.concatenate([np.linspace(0, 2, 1001), np.exp(np.linspace(-12, 6, 500))])
    x = x[x <= 448]
    ref = torch.tensor(x, dtype=torch.float32).to(torch.float8_e4m3fn).double().numpy()
    assert np.array_equal(_e4m3_round(x.astype(np.float32).astype(np.float64)), ref)
