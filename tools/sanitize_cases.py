"""Small forward/backward cases over every code path (fixed, GQA split, deterministic,
N_q != N_k, varlen with empty sequences, FP8, the CTA-pair forward and backward) for
compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_08691_b200 as fa2

torch.manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16)
for d in (64, 128):
    for causal in (False, True):
        q, k, v, do = mk(2, 4, 300, d), mk(2, 2, 300, d), mk(2, 2, 300, d), mk(2, 4, 300, d)
        o, l = fa2.forward(q, k, v, causal=causal)
        fa2.backward(q, k, v, o, l, do, causal=causal)                       # GQA split
        fa2.backward(q, k, v, o, l, do, causal=causal, deterministic=True)
        q2, do2 = mk(1, 2, 200, d), mk(1, 2, 200, d)
        k2, v2 = mk(1, 2, 333, d), mk(1, 2, 333, d)
        o2, l2 = fa2.forward(q2, k2, v2, causal=causal)                      # N_q != N_k
        fa2.backward(q2, k2, v2, o2, l2, do2, causal=causal)
        cu_q = torch.tensor([0, 100, 100, 357, 400], dtype=torch.int32, device="cuda")
        cu_k = torch.tensor([0, 300, 400, 529, 529], dtype=torch.int32, device="cuda")
        qv, dov = mk(400, 4, d), mk(400, 4, d)
        kv_, vv = mk(529, 2, d), mk(529, 2, d)
        ov, lv = fa2.forward_varlen(qv, kv_, vv, cu_q, cu_k, 257, 300, causal=causal)
        fa2.backward_varlen(qv, kv_, vv, ov, lv, dov, cu_q, cu_k, 257, 300, causal=causal)
    # causal square shapes long enough for the balanced tile schedule to reorder tiles
    q3, k3, v3, do3 = (mk(1, 3, 1500, d) for _ in range(4))
    o3, l3 = fa2.forward(q3, k3, v3, causal=True)
    fa2.backward(q3, k3, v3, o3, l3, do3, causal=True)
    # square MHA shapes: the CTA-pair forward (d = 128, causal and not) and the CTA-pair backward
    # (d = 128, causal and not), ragged (700 = 2 pair key blocks + a 188-row tail)
    for causal in (False, True):
        q4, k4, v4, do4 = (mk(1, 2, 700, d) for _ in range(4))
        o4, l4 = fa2.forward(q4, k4, v4, causal=causal)
        fa2.backward(q4, k4, v4, o4, l4, do4, causal=causal)
    if d == 128:
        q8, k8, v8 = (mk(1, 2, 300, 128).to(torch.float8_e4m3fn) for _ in range(3))
        fa2.forward_fp8(q8, k8, v8, causal=True)
torch.cuda.synchronize()
print("sanitize cases done")
