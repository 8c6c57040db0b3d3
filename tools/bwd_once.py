"""One forward + a few backward passes at the bench workload (PS-128 N=8k, B=2, H=16),
for ncu captures of a single kernel: python tools/bwd_once.py [causal] [d]."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2
causal = len(sys.argv) > 1 and sys.argv[1] == "1"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
H = 16 if d == 128 else 32
B, N = 2, 8192
q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = fa2.forward(q, k, v, causal=causal)
for _ in range(3):
    fa2.backward(q, k, v, o, lse, do, causal=causal)
torch.cuda.synchronize()
print("ok")
