"""Print the forward kernel's clock64 timeline for CTA 0's first tile (debug build hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_08691_b200 as fa2

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
H = 16 if d == 128 else 32
B, N = 2, 8192
q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
tr = torch.zeros(16384, dtype=torch.int64, device="cuda")
for _ in range(3):
    fa2.forward(q, k, v, causal=causal)
fa2.lib().fa2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
fa2.forward(q, k, v, causal=causal)
fa2.lib().fa2_debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().view(-1, 64)
ev = lambda e, w: t[e * 2 + w]
base = int(ev(0, 0)[0])
names = ["s_full_ok", "max_done", "exp_done", "p_arrive", "mma_p_ok", "mma_S_issued"]
print("j  | " + " | ".join(f"{n}0 {n}1" for n in names))
for j in range(0, 64, 4):
    row = []
    for e in range(6):
        for w in range(2):
            x = int(ev(e, w)[j])
            row.append(f"{x - base:7d}" if x else "      -")
    print(f"{j:2d} | " + " ".join(row))
# per-iteration averages (steady state j in [8, 56))
import statistics
def dd(a, b, w1, w2, lag=0):
    return statistics.mean(int(ev(b, w2)[j + lag]) - int(ev(a, w1)[j]) for j in range(8, 56))
print("period (s_full_ok0 j -> j+1):", statistics.mean(int(ev(0, 0)[j + 1]) - int(ev(0, 0)[j]) for j in range(8, 56)))
print("softmax0: s_full->max", dd(0, 1, 0, 0), " max->exp", dd(1, 2, 0, 0), " exp->arrive", dd(2, 3, 0, 0))
print("arrive0 -> mma sees p0:", dd(3, 4, 0, 0), "  mma p0 -> S0(j+1) issued:", dd(4, 5, 0, 0))
print("S0(j+1) issued -> softmax0 s_full(j+1):", dd(5, 0, 0, 0, lag=1))
