"""Forward TFLOP/s over the paper sweep (N = 512..8k, B = 16k/N, hidden 2048) for the
library selected by FA2_LIB_PATH (A/B builds)."""
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
for d, H in ((128, 16), (64, 32)):
    for N in (512, 1024, 2048, 4096, 8192):
        B = 16384 // N
        q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        for causal in (False, True):
            fl = 4.0 * N * N * d * H * B / (2 if causal else 1)
            res[f"d{d}_N{N}_c{int(causal)}"] = round(fl / tm(lambda: fa2.forward(q, k, v, causal=causal)) / 1e9, 1)
print(json.dumps(res))
