"""Deterministic backward (include/fa2.h fa2_backward_deterministic):
parity with the fp64 oracle (same tolerances as fa2_backward), bitwise
reproducibility across runs, and agreement with the arrival-order backward.
Covers both schedules: the cyclic one (key blocks per head <= #SMs) and the
ascending fallback (a head with more key blocks than SMs)."""
import numpy as np
import pytest
import torch

import paper_2307_08691_b200 as fa2
import workloads as W
from oracle import ref_attention as R
from tests.gpu_util import TOL, grad_floor, grad_ok, scale_for, to_np

pytestmark = pytest.mark.gpu


def _fwd_bwd(q, k, v, do, causal, sc, deterministic, reps=1):
    qc, kc, vc, doc = q.cuda(), k.cuda(), v.cuda(), do.cuda()
    o, lse = fa2.forward(qc, kc, vc, causal=causal, softmax_scale=sc)
    outs = [fa2.backward(qc, kc, vc, o, lse, doc, causal=causal, softmax_scale=sc, deterministic=deterministic)
            for _ in range(reps)]
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(1, 2, 1000, 128), (2, 3, 300, 64), (1, 1, 129, 128), (1, 2, 1, 64),
                                   (2, 4, 2, 520, 128)], ids=lambda s: "x".join(map(str, s)))
def test_deterministic_parity(shape, causal, dtype):
    if len(shape) == 5:
        B, H, Hkv, N, d = shape
    else:
        (B, H, N, d), Hkv = shape, shape[1]
    q, _, _, do = W.qkv(B, H, N, d, dtype, seed=900 + N + d)
    k = W.randn((B, Hkv, N, d), 950 + N, dtype)
    v = W.randn((B, Hkv, N, d), 951 + N, dtype)
    sc = scale_for(d)
    (dq, dk, dv), = _fwd_bwd(q, k, v, do, causal, sc, True)
    if Hkv == H:
        gq, gk, gv, _ = R.backward(to_np(q), to_np(k), to_np(v), to_np(do), sc, causal)
    else:
        gq, gk, gv = R.backward_gqa(to_np(q), to_np(k), to_np(v), to_np(do), sc, causal)
    fl = grad_floor(gq, gk, gv)
    for name, g, ref in (("dq", dq, gq), ("dk", dk, gk), ("dv", dv, gv)):
        ok, err, lim = grad_ok(g, ref, dtype, fl, degenerate=(N == 1))   # N = 1: dQ = dK = 0 exactly
        assert ok, f"{name}: err {err} > {lim}"


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("d", [64, 128])
def test_deterministic_bitwise(causal, d):
    """Many key blocks per dQ tile (N=4096: 32), several heads -> many CTAs race on
    every dQ tile; three runs must agree bit for bit, and with the arrival-order
    backward to within rounding of the summation order."""
    B, H, N = 2, 6, 4096
    q, k, v, do = W.qkv(B, H, N, d, "bf16", seed=77 + d)
    sc = scale_for(d)
    runs = _fwd_bwd(q, k, v, do, causal, sc, True, reps=3)
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert torch.equal(a, b)
    base = _fwd_bwd(q, k, v, do, causal, sc, False)[0]
    if causal:   # same query-tile order -> dK, dV (accumulated on chip) are identical
        assert torch.equal(base[1], runs[0][1]) and torch.equal(base[2], runs[0][2])
    for a, b in zip(base, runs[0]):   # non-causal visits query tiles in rotated order: rounding only
        rel = float((a.float() - b.float()).abs().max()) / float(a.float().abs().max())
        assert rel <= 2 ** -6, rel


@pytest.mark.parametrize("d", [64, 128])
def test_deterministic_fallback_schedule(d):
    """N = 149*128: 149 key blocks > 148 SMs (d = 64, one-SM kernel) and 75 key-block pairs
    > 74 CTA pairs (d = 128, CTA-pair kernel) -> the ascending-order schedule.  Bitwise
    repeatable, and sampled rows match the oracle."""
    B, H, N = 1, 1, 149 * 128
    q, k, v, do = W.qkv(B, H, N, d, "bf16", seed=31)
    sc = scale_for(d)
    runs = _fwd_bwd(q, k, v, do, True, sc, True, reps=2)
    for a, b in zip(runs[0], runs[1]):
        assert torch.equal(a, b)
    dq, dk, dv = runs[0]
    rows = np.array([0, 1, 127, 128, 5000, N // 2, N - 129, N - 1])
    f64 = lambda t: t.double().numpy()
    sm = R.backward_sampled_head(f64(q[0, 0]), f64(k[0, 0]), f64(v[0, 0]), f64(do[0, 0]), sc, True,
                                 dq_rows=rows, dkv_cols=rows, rows_per_chunk=1024)
    got = {"dq": dq[0, 0, rows], "dk": dk[0, 0, rows], "dv": dv[0, 0, rows]}
    for x in ("dq", "dk", "dv"):   # not degenerate: plain rule R15
        err = float(np.max(np.abs(got[x].double().cpu().numpy() - sm[x])))
        lim = TOL["bf16"]["grad"] * float(np.max(np.abs(sm[x])))
        assert err <= lim, (x, err, lim)
