"""A few forward launches at the paper shape for ncu captures: python tools/fwd_once.py d causal [N]."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2
d, causal = int(sys.argv[1]), sys.argv[2] == "1"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
B, H = max(1, 16384 // N), 2048 // d
q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(3):
    fa2.forward(q, k, v, causal=causal)
torch.cuda.synchronize()
print("ok")
