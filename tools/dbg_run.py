"""Quick GPU diagnostics: forward/backward on small shapes vs the oracle, printing errors."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_08691_b200 as fa2
import workloads as W
from oracle import ref_attention as R

f64 = lambda t: t.double().cpu().numpy()
for (B, H, N, d) in [(1, 1, 128, 64), (1, 1, 128, 128), (1, 2, 300, 64), (1, 2, 600, 128)]:
    for causal in (False, True):
        sc = 1 / math.sqrt(d)
        q, k, v, do = W.qkv(B, H, N, d, "bf16", seed=1)
        qc, kc, vc, doc = (t.cuda() for t in (q, k, v, do))
        o, lse = fa2.forward(qc, kc, vc, causal=causal, softmax_scale=sc)
        torch.cuda.synchronize()
        o_ref, l_ref = R.forward(f64(q), f64(k), f64(v), sc, causal)
        eo = np.abs(f64(o) - o_ref); el = np.abs(f64(lse) - l_ref)
        print(f"FWD B{B} H{H} N{N} d{d} c{int(causal)}: O err {eo.max():.3e} (argmax {np.unravel_index(eo.argmax(), eo.shape)}) L err {el.max():.3e}", flush=True)
        dq, dk, dv = fa2.backward(qc, kc, vc, o, lse, doc, causal=causal, softmax_scale=sc)
        torch.cuda.synchronize()
        g = R.backward(f64(q), f64(k), f64(v), f64(do), sc, causal)
        for nm, a, r in zip(("dq", "dk", "dv"), (dq, dk, dv), g[:3]):
            e = np.abs(f64(a) - r)
            print(f"   BWD {nm}: err {e.max():.3e} rel {e.max()/np.abs(r).max():.3e} argmax {np.unravel_index(e.argmax(), e.shape)}", flush=True)
