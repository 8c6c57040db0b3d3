"""Per-CTA block timeline of the forward's first work tile (every CTA; debug trace hook):
period per key block, phase offset between the two softmax warpgroups, exp-phase length.
usage: python tools/phase_trace_fwd.py D CAUSAL [N]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2307_08691_b200 as fa2

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
H = 16 if d == 128 else 32
B = 16384 // N
q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(5):
    fa2.forward(q, k, v, causal=causal)
tr = torch.zeros(65536 + 148 * 8 * 2 * 64, dtype=torch.int64, device="cuda")
fa2.lib().fa2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
fa2.forward(q, k, v, causal=causal)
fa2.lib().fa2_debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy()[65536:].reshape(148, 8, 2, 64).astype(np.float64)
J = slice(8, 56)
rows = []
for c in range(148):
    e3 = t[c, 3]
    if not (e3[0, 8:57] > 0).all() or not (e3[1, 8:57] > 0).all():
        continue
    per = np.mean(np.diff(e3[0, 8:57]))
    ph = np.mean(((e3[1, J] - e3[0, J]) % per) / per)
    expl = [np.mean(t[c, 2, w, J] - t[c, 1, w, J]) for w in (0, 1)]
    wait_s = [np.mean(t[c, 1, w, 9:57] - t[c, 3, w, 8:56]) for w in (0, 1)]   # arrive(j) -> top of j+1
    rows.append((per, ph, expl[0], expl[1], wait_s[0], wait_s[1], c))
rows.sort()
print(f"{len(rows)} CTAs traced; columns: period, phase(wg1-wg0)/period, exp0, exp1, arrive->next top 0/1, cta")
for r in rows[:8] + [None] + rows[-8:]:
    print("  ..." if r is None else "  %6.0f  %.2f  %6.0f %6.0f  %6.0f %6.0f  cta %d" % r)
per = np.array([r[0] for r in rows]); ph = np.array([r[1] for r in rows])
print("corr(period, |phase-0.5|) = %.2f" % np.corrcoef(per, np.abs(ph - 0.5))[0, 1])
