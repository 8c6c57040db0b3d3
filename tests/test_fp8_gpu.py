"""FP8 forward (fa2_forward_fp8) vs the fp64 oracle.

The represented inputs descale_x * x8 (x8 in E4M3) are exact in float64, so the
expected O and L are the plain definition on them (oracle.forward_gqa).  The
kernel rounds P~ to E4M3 before P~V (R25), so O is checked against the
oracle's per-element bound fp8_pv_error_bound plus bf16 output rounding (half an
ulp) and 2^-11 * sum_j P_ij |V_jc| for the fp32 exp2 approximations; L (summed
from fp32 P~) keeps the bf16/fp16 tolerance 1e-3."""
import numpy as np
import pytest
import torch

import paper_2307_08691_b200 as fa2
import workloads as W
from oracle import ref_attention as R
from tests.fp8_bound import fp8_pv_error_bound
from tests.gpu_util import TOL, half_ulp, scale_for

pytestmark = pytest.mark.gpu


def _quant(x, amax_target=224.0):
    """x (fp32) -> (E4M3 tensor, descale) with max |x| / descale = amax_target."""
    descale = float(x.abs().max()) / amax_target
    return (x / descale).to(torch.float8_e4m3fn), descale


def _check(o, lse, q8, k8, v8, dq, dk, dv, sc, causal):
    qd = q8.double().numpy() * dq
    kd = k8.double().numpy() * dk
    vd = v8.double().numpy() * dv
    o_ref, l_ref = R.forward_gqa(qd, kd, vd, sc, causal)
    B, H, N, d = qd.shape
    group = H // kd.shape[1]
    og = o.double().cpu().numpy()
    for b in range(B):
        for h in range(H):
            bound = fp8_pv_error_bound(qd[b, h], kd[b, h // group], vd[b, h // group], sc, causal)
            p, _, _ = R.softmax_rows(R.scores(qd[b, h], kd[b, h // group], sc, causal))
            slack = 2.0 ** -11 * (p @ np.abs(vd[b, h // group]))
            err = np.abs(og[b, h] - o_ref[b, h]) - half_ulp(o_ref[b, h], "bf16")
            assert np.all(err <= bound + slack), float(np.max(err - bound - slack))
    assert float(np.max(np.abs(lse.cpu().numpy() - l_ref))) <= TOL["bf16"]["L"]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (1, 2, 2, 129), (2, 2, 1, 256), (1, 4, 2, 1000), (1, 1, 1, 2048)],
                         ids=lambda s: "x".join(map(str, s)))
def test_fp8_forward_parity(shape, causal):
    B, H, Hkv, N = shape
    d = 128
    q8, dq = _quant(W.randn((B, H, N, d), 400 + N, "fp32"))
    k8, dk = _quant(W.randn((B, Hkv, N, d), 401 + N, "fp32"))
    v8, dv = _quant(W.randn((B, Hkv, N, d), 402 + N, "fp32"))
    sc = scale_for(d)
    o, lse = fa2.forward_fp8(q8.cuda(), k8.cuda(), v8.cuda(), dq, dk, dv, causal=causal, softmax_scale=sc)
    torch.cuda.synchronize()
    assert o.dtype == torch.bfloat16 and torch.isfinite(o.float()).all()
    _check(o, lse, q8, k8, v8, dq, dk, dv, sc, causal)


def test_fp8_matches_bf16_path_on_representable_inputs():
    """Inputs whose values are exactly representable in both E4M3 and bf16 (descale 1):
    the FP8 path and the bf16 path compute the same S, so their O differ only by the
    E4M3 rounding of P~ (bounded as above) -- and L agrees to fp32 rounding."""
    B, H, N, d = 1, 2, 512, 128
    x = [W.randn((B, H, N, d), 410 + i, "fp32").to(torch.float8_e4m3fn) for i in range(3)]
    o8, l8 = fa2.forward_fp8(*(t.cuda() for t in x), causal=True)
    ob, lb = fa2.forward(*(t.to(torch.bfloat16).cuda() for t in x), causal=True)
    torch.cuda.synchronize()
    assert float((l8 - lb).abs().max()) <= 1e-4
    _check(o8, l8, *x, 1.0, 1.0, 1.0, scale_for(d), True)


def test_fp8_errors():
    z = torch.zeros(1, 1, 128, 64, dtype=torch.float8_e4m3fn, device="cuda")
    with pytest.raises(fa2.FA2Error):
        fa2.forward_fp8(z, z, z)                       # d = 64 unsupported
    z = torch.zeros(1, 1, 128, 128, dtype=torch.float8_e4m3fn, device="cuda")
    with pytest.raises(fa2.FA2Error):
        fa2.forward_fp8(z, z, z, descale_q=0.0)        # descale must be > 0
    with pytest.raises(fa2.FA2Error):
        fa2.forward_fp8(z.to(torch.bfloat16), z, z)    # dtype
