"""clock64 timeline of the CTA-pair d=128 backward (FA2_BWD_PAIR=1), CTA 0, query steps 6-55."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FA2_BWD_PAIR"] = "1"
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
    return round(statistics.mean(int(t[b][h + lag]) - int(t[a][h]) for h in rng), 1)
print("period (compute s_full seen):", avg(0, 0, 1))
print("compute: P phase s_full->p_ready", avg(0, 1), "(exps", avg(0, 15), ") | p_ready->dp_full seen", avg(1, 2),
      "| dS: math", avg(2, 11), " slot/staging waits", avg(11, 12), " sts+fence+wait st", avg(12, 13),
      " arrive", avg(13, 3), "| ds_ready->next s_full seen", avg(3, 0, 1))
print("mma: ds_ready seen -> dK+dP issued, s_consumed", avg(7, 8), "| exchange wait + dQ issue", avg(8, 5),
      "| -> p_ready(x+1) seen", avg(5, 4, 1), "| dV + S issue", avg(4, 6), "| -> ds_ready seen", avg(6, 7))
print("dQ warps: dq_full seen -> read out", avg(9, 10), "| reduce issue", avg(10, 16), "| -> next dq_full", avg(16, 9, 1))
print("exchange (CTA 0 -> 1): ds_ready(x) -> xs_full seen", avg(3, 17), "| ds_free wait", avg(17, 18),
      "| copy read done", avg(18, 19), "| CTA 1 -> 0 landed (dsx_full seen) after copy issue", avg(18, 20),
      "| dQ issued after landing", avg(20, 5))
print("mma in issue_dq: dsx_full seen after event 8", avg(8, 21), "| dsx_ready (relay) seen after dsx_full", avg(21, 22),
      "| dQ MMAs issued after both", avg(22, 5))
