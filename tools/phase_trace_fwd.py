"""Per-CTA block timeline of the forward's first work tile (every CTA; debug trace hook):
period per key block, phase offset between the two softmax warpgroups, and the softmax
sub-phases (pair kernel events: 0 S ready, 1 row max done, 6 P~ buffer free / O rescaled,
7 ping-pong wait done, 2 exponentials done, 3 P~ handed over).
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
J = slice(8, 40)  # steady-state blocks of the first tile
rows = []
sub = {w: [] for w in (0, 1)}
for c in range(148):
    e3 = t[c, 3]
    if not (e3[0, 8:41] > 0).all() or not (e3[1, 8:41] > 0).all():
        continue
    per = np.mean(np.diff(e3[0, 8:41]))
    ph = np.mean(((e3[1, J] - e3[0, J]) % per) / per)
    rows.append((per, ph, c))
    for w in (0, 1):
        ev = lambda e, lag=0: t[c, e, w, 8 + lag:40 + lag]
        sub[w].append([np.mean(ev(0, 1) - ev(3)),   # arrive(j) -> S(j+1) seen
                       np.mean(ev(1) - ev(0)),       # S seen -> max done
                       np.mean(ev(6) - ev(1)),       # -> P~ buffer free (o_done) / rescale
                       np.mean(ev(7) - ev(6)),       # ping-pong wait
                       np.mean(ev(2) - ev(7)),       # exponentials
                       np.mean(ev(3) - ev(2))])      # fence + arrive
rows.sort()
print(f"{len(rows)} CTAs; period min {rows[0][0]:.0f} median {rows[len(rows) // 2][0]:.0f} max {rows[-1][0]:.0f}; "
      f"phase (wg1 - wg0) / period median {np.median([r[1] for r in rows]):.2f}")
for w in (0, 1):
    m = np.mean(np.array(sub[w]), axis=0) if sub[w] else np.zeros(6)
    print(f"wg{w} sub-phases (cycles): arrive->S seen {m[0]:.0f} | ld+max {m[1]:.0f} | o_done/rescale {m[2]:.0f} | "
          f"pp wait {m[3]:.0f} | exps {m[4]:.0f} | fence+arrive {m[5]:.0f}")
# MMA side (leader CTAs; issuer i = sub-tile i): P~ handed over -> issuer sees it (ev3 -> ev4),
# P~V issued -> softmax sees it complete (ev4[j] -> ev6[j + 1]), S(j+1) issued -> S seen (ev5 -> ev0)
lat = {w: [] for w in (0, 1)}
for c in range(0, 148, 2):
    for w in (0, 1):
        e = lambda ev, lag=0: t[c, ev, w, 8 + lag:40 + lag]
        if not (e(4) > 0).all() or not (e(6, 1) > 0).all():
            continue
        lat[w].append([np.mean(e(4) - e(3)), np.mean(e(6, 1) - e(4)), np.mean(e(0, 1) - e(5, 1))])
for w in (0, 1):
    if lat[w]:
        m = np.mean(np.array(lat[w]), axis=0)
        print(f"sub-tile {w} (leader CTAs): p_full -> issuer sees {m[0]:.0f} | P~V issued -> o_done seen by softmax "
              f"{m[1]:.0f} | S issued -> s_full seen {m[2]:.0f}")
