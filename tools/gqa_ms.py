"""GQA/MQA backward TFLOP/s (B=2, H=32, N=8k, d=128) for the checkout in cwd."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2
res = {}
for hkv in (8, 4, 1):
    for causal in (False, True):
        B, H, N, d = 2, 32, 8192, 128
        mk = lambda h: torch.randn(B, h, N, d, device="cuda", dtype=torch.bfloat16)
        q, k, v, do = mk(H), mk(hkv), mk(hkv), mk(H)
        o, lse = fa2.forward(q, k, v, causal=causal)
        ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
        f = lambda: fa2.backward(q, k, v, o, lse, do, causal=causal, workspace=ws)
        for _ in range(3): f()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        fl = 2.5 * 4.0 * N * N * d * H * B / (2 if causal else 1)
        res[f"hkv{hkv}_c{int(causal)}"] = round(fl / (s.elapsed_time(e) / 10) / 1e9, 1)
print(json.dumps(res))
