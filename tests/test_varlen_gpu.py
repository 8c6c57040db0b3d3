"""N_q != N_k (fa2_forward_ex / fa2_backward_ex) and packed variable-length
batches (fa2_forward_varlen / fa2_backward_varlen), vs the fp64
oracle's *_general / *_varlen functions (bottom-right causal alignment R22;
rows that see no key: O = 0, L = -inf, R23).  Same tolerances as the square
path (BASELINE north_star; R14, R15)."""
import numpy as np
import pytest
import torch

import paper_2307_08691_b200 as fa2
import workloads as W
from oracle import ref_attention as R
from tests.gpu_util import TOL, grad_floor, grad_ok, max_abs, o_excess, scale_for, to_np

pytestmark = pytest.mark.gpu


def _lse_ok(got, ref, dtype):
    got = np.asarray(got, dtype=np.float64)
    assert np.array_equal(np.isneginf(got), np.isneginf(ref)), "rows without keys must have L = -inf"
    fin = np.isfinite(ref)
    assert np.all(np.isfinite(got[fin]))
    assert float(np.max(np.abs(got[fin] - ref[fin]), initial=0.0)) <= TOL[dtype]["L"]


def _grads_ok(got, ref, dtype):
    fl = grad_floor(*ref)
    for name, g, r in zip(("dq", "dk", "dv"), got, ref):
        assert torch.isfinite(g.float()).all(), name
        ok, err, lim = grad_ok(g, r, dtype, fl)
        assert ok, f"{name}: err {err} > {lim}"


FIXED = [  # B, H, H_kv, N_q, N_k, d
    (2, 2, 2, 100, 300, 64),
    (1, 2, 1, 300, 100, 128),
    (1, 3, 3, 257, 129, 64),
    (2, 4, 2, 1000, 517, 128),
    (1, 1, 1, 128, 1000, 128),
]


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", FIXED, ids=lambda s: "x".join(map(str, s)))
def test_rectangular_parity(shape, causal, dtype):
    B, H, Hkv, Nq, Nk, d = shape
    q = W.randn((B, H, Nq, d), 300 + Nq, dtype)
    k = W.randn((B, Hkv, Nk, d), 301 + Nk, dtype)
    v = W.randn((B, Hkv, Nk, d), 302 + Nk, dtype)
    do = W.randn((B, H, Nq, d), 303 + Nq, dtype)
    sc = scale_for(d)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = fa2.forward(qc, kc, vc, causal=causal, softmax_scale=sc)
    dq, dk, dv = fa2.backward(qc, kc, vc, o, lse, doc, causal=causal, softmax_scale=sc)
    torch.cuda.synchronize()
    # oracle: the packed varlen oracle on the same data (one sequence per batch entry)
    cu_q = np.arange(B + 1) * Nq
    cu_k = np.arange(B + 1) * Nk
    pk = lambda t: to_np(t).transpose(0, 2, 1, 3).reshape(-1, t.shape[1], d)
    o_ref, l_ref = R.forward_varlen(pk(q), pk(k), pk(v), cu_q, cu_k, sc, causal)
    gq, gk, gv = R.backward_varlen(pk(q), pk(k), pk(v), pk(do), cu_q, cu_k, sc, causal)
    unpk = lambda a, n, h: a.reshape(B, n, h, d).transpose(0, 2, 1, 3)
    assert o_excess(o.cpu(), unpk(o_ref, Nq, H), dtype) <= TOL[dtype]["O"]
    _lse_ok(lse.cpu().numpy(), l_ref.reshape(H, B, Nq).transpose(1, 0, 2), dtype)
    _grads_ok((dq, dk, dv), (unpk(gq, Nq, H), unpk(gk, Nk, Hkv), unpk(gv, Nk, Hkv)), dtype)


VARLEN = [  # (cu_q, cu_k): empty query sequence, N_q > N_k, N_q < N_k, empty key sequence, long sequence
    ([0, 100, 100, 357, 1357, 1400], [0, 300, 400, 529, 1529, 1529]),
    ([0, 1, 130, 700], [0, 128, 129, 900]),
]


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("case", [0, 1])
def test_varlen_parity(case, d, causal, dtype):
    cu_q, cu_k = VARLEN[case]
    H, Hkv = 4, 2
    Tq, Tk = cu_q[-1], cu_k[-1]
    q = W.randn((Tq, H, d), 310 + case, dtype)
    k = W.randn((Tk, Hkv, d), 311 + case, dtype)
    v = W.randn((Tk, Hkv, d), 312 + case, dtype)
    do = W.randn((Tq, H, d), 313 + case, dtype)
    sc = scale_for(d)
    cq = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
    ck = torch.tensor(cu_k, dtype=torch.int32, device="cuda")
    mq, mk = int(np.max(np.diff(cu_q))), int(np.max(np.diff(cu_k)))
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = fa2.forward_varlen(qc, kc, vc, cq, ck, mq, mk, causal=causal, softmax_scale=sc)
    dq, dk, dv = fa2.backward_varlen(qc, kc, vc, o, lse, doc, cq, ck, mq, mk, causal=causal, softmax_scale=sc)
    torch.cuda.synchronize()
    o_ref, l_ref = R.forward_varlen(to_np(q), to_np(k), to_np(v), cu_q, cu_k, sc, causal)
    gq, gk, gv = R.backward_varlen(to_np(q), to_np(k), to_np(v), to_np(do), cu_q, cu_k, sc, causal)
    assert o_excess(o.cpu(), o_ref, dtype) <= TOL[dtype]["O"]
    _lse_ok(lse.cpu().numpy(), l_ref, dtype)
    _grads_ok((dq, dk, dv), (gq, gk, gv), dtype)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_varlen_equal_lengths_match_fixed_layout(causal, d):
    """Equal lengths: the packed path computes what the [B,H,N,d] path does.  Causal
    d = 64: the same one-SM forward kernel, forward bitwise.  d = 128 (causal and not): the
    fixed layout runs the CTA-pair forward, whose exponential split (2 of 16 pairs on the FMA
    pipe instead of 4; masked blocks all on MUFU in both) and key-block split over the pair
    round P~ differently, so forward to within a bf16 rounding step (non-causal d = 64: same
    kernel, compared the same way).  Backward up to the dQ summation order (and the forward
    difference)."""
    B, H, N = 3, 2, 300
    q, k, v, do = W.qkv(B, H, N, d, "bf16", seed=320)
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = fa2.forward(qc, kc, vc, causal=causal)
    dq, dk, dv = fa2.backward(qc, kc, vc, o, lse, doc, causal=causal)
    pk = lambda t: t.transpose(1, 2).reshape(B * N, H, d).contiguous()
    cu = torch.arange(B + 1, dtype=torch.int32, device="cuda") * N
    o2, lse2 = fa2.forward_varlen(pk(qc), pk(kc), pk(vc), cu, cu, N, N, causal=causal)
    dq2, dk2, dv2 = fa2.backward_varlen(pk(qc), pk(kc), pk(vc), o2, lse2, pk(doc), cu, cu, N, N, causal=causal)
    torch.cuda.synchronize()
    if causal and d == 64:
        assert torch.equal(pk(o), o2)
        assert torch.equal(lse.transpose(0, 1).reshape(H, B * N), lse2)
    else:
        diff = (pk(o).float() - o2.float()).abs()
        assert bool((diff <= 2 ** -7 * o2.float().abs() + 1e-3).all()), float(diff.max())
        assert float((lse.transpose(0, 1).reshape(H, B * N) - lse2).abs().max()) <= 1e-4
    for a, b in ((dq, dq2), (dk, dk2), (dv, dv2)):
        rel = float((pk(a).float() - b.float()).abs().max()) / float(b.float().abs().max())
        assert rel <= 2 ** -6, rel


def test_varlen_deterministic_bitwise():
    cu_q, cu_k = [0, 700, 700, 2000, 2100], [0, 500, 900, 2200, 2300]
    H, Hkv, d = 4, 4, 64
    q = W.randn((cu_q[-1], H, d), 330, "bf16").cuda()
    k = W.randn((cu_k[-1], Hkv, d), 331, "bf16").cuda()
    v = W.randn((cu_k[-1], Hkv, d), 332, "bf16").cuda()
    do = W.randn((cu_q[-1], H, d), 333, "bf16").cuda()
    cq = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
    ck = torch.tensor(cu_k, dtype=torch.int32, device="cuda")
    o, lse = fa2.forward_varlen(q, k, v, cq, ck, 1300, 1300, causal=True)
    runs = [fa2.backward_varlen(q, k, v, o, lse, do, cq, ck, 1300, 1300, causal=True, deterministic=True)
            for _ in range(3)]
    torch.cuda.synchronize()
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert torch.equal(a, b)
