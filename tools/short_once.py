"""Short-sequence launches for ncu captures: python tools/short_once.py d causal [bwd]
(PS shapes: N = 512, B = 32, H = 2048 / d)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2
d, causal = int(sys.argv[1]), sys.argv[2] == "1"
bwd = len(sys.argv) > 3 and sys.argv[3] == "bwd"
N, B, H = 512, 32, 2048 // d
q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
for _ in range(3):
    o, lse = fa2.forward(q, k, v, causal=causal)
    if bwd:
        fa2.backward(q, k, v, o, lse, do, causal=causal)
torch.cuda.synchronize()
print("ok")
