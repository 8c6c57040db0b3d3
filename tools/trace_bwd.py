"""Print the backward kernel's clock64 timeline (CTA 0, first 64 query tiles) via fa2_debug_set_trace."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_08691_b200 as fa2

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
H = 16 if d == 128 else 32
B, N = 2, 8192
q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = fa2.forward(q, k, v, causal=causal)
for _ in range(2):
    fa2.backward(q, k, v, o, lse, do, causal=causal)
tr = torch.zeros(16384, dtype=torch.int64, device="cuda")
fa2.lib().fa2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
fa2.backward(q, k, v, o, lse, do, causal=causal)
fa2.lib().fa2_debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().view(-1, 64)
names = ["c:s_full", "c:s_cons", "c:ds_empty", "c:ds_ready", "m:S_iss", "m:ds_rdy", "m:dQ_iss", "q:dq_full", "q:red_iss", "m:S_start"]
base = int(t[0][0])
print("h  | " + " ".join(f"{n:>10s}" for n in names))
for h in range(0, 64, 7):
    print(f"{h:2d} | " + " ".join(f"{(int(t[e][h]) - base) if int(t[e][h]) else 0:10d}" for e in range(10)))
rng = range(8, 60)
def avg(a, b, lag=0):
    return statistics.mean(int(t[b][h + lag]) - int(t[a][h]) for h in rng)
print("period (compute s_full):", avg(0, 0, 1))
print("compute: s_full -> ds_ready arrive", avg(0, 3))
print("mma: ds_ready arrive -> seen", avg(3, 5), "  grads issue", avg(5, 6))
print("mma: dQ issued(h) -> S/dP(h+2) issued", avg(6, 4, 2), "   S/dP(h) issued -> compute sees s_full(h)", avg(4, 0))
print("dq: dQ issued -> dq_full seen", avg(6, 7), "  dq_full -> reduce issued", avg(7, 8))
