"""Forward TFLOP/s (bf16 d=128/64 and FP8 d=128, N=8k, causal and not) for the checkout in cwd."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2

def tm(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

res = {}
for kind, d, H in (("bf16", 128, 16), ("bf16", 64, 32), ("fp8", 128, 16)):
    for causal in (False, True):
        B, N = 2, 8192
        mk = lambda: torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
        q, k, v = mk(), mk(), mk()
        if kind == "fp8":
            q, k, v = (t.to(torch.float8_e4m3fn) for t in (q, k, v))
            fn = lambda: fa2.forward_fp8(q, k, v, causal=causal)
        else:
            fn = lambda: fa2.forward(q, k, v, causal=causal)
        fl = 4.0 * N * N * d * H * B / (2 if causal else 1)
        res[f"{kind}_d{d}_c{int(causal)}"] = round(fl / tm(fn) / 1e9, 1)
print(json.dumps(res))
