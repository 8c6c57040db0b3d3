"""clock64 timeline of the d=128 backward kernel (CTA 0, first 64 query tiles)."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_08691_b200 as fa2
causal = len(sys.argv) > 1 and sys.argv[1] == "1"
B, H, N, d = 2, 16, 8192, 128
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
rng = range(6, 56)
def avg(a, b, lag=0):
    return statistics.mean(int(t[b][h + lag]) - int(t[a][h]) for h in rng)
print("period (P warps s_full):", avg(0, 0, 1))
print("P phase: s_full->p_ready", avg(0, 1), "  dS phase: dp_full->dst_ready", avg(2, 3))
print("mma: p_ready->seen", avg(1, 4), " dV+dP issue", avg(4, 5), " S(x+1) issue", avg(5, 6),
      " ->dst_ready seen", avg(6, 7), " dK+dQ issue", avg(7, 8), " dQ issued -> next p_ready seen", avg(8, 4, 1))
print("dQ warps: dq_full seen->dq_empty", avg(9, 10), " dq_empty->rounds issued", avg(10, 16),
      " rounds issued->next dq_full seen", avg(16, 9, 1), " dQ issued(mma)->dq_full seen", avg(8, 9))
print("P sub-phases: s_full->exps done", avg(0, 15), " exps->p_ready", avg(15, 1))
print("dS sub-phases: dp_full->math done", avg(2, 11), " ->tmem st+sts issued", avg(11, 12), " ->wait st", avg(12, 13),
      " ->fence.proxy", avg(13, 14), " ->arrive", avg(14, 3))
