"""Backward TFLOP/s, arrival-order vs deterministic, at the bench workload and a causal case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_08691_b200 as fa2

for (B, H, N, d, causal) in [(2, 16, 8192, 128, False), (2, 16, 8192, 128, True), (4, 32, 4096, 64, False),
                             (1, 16, 32768, 128, True)]:
    q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o, lse = fa2.forward(q, k, v, causal=causal)
    ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
    res = {}
    for det in (False, True):
        for _ in range(3):
            fa2.backward(q, k, v, o, lse, do, causal=causal, workspace=ws, deterministic=det)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fa2.backward(q, k, v, o, lse, do, causal=causal, workspace=ws, deterministic=det)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        flops = 2.5 * 4.0 * N * N * d * H * B / (2 if causal else 1)   # paper count
        res["det" if det else "atomic"] = round(flops / ms / 1e9, 1)
    print((B, H, N, d, causal), res, flush=True)
