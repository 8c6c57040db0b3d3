"""Per-work-tile timeline of the CTA-pair backward (debug hook): for every CTA's first 32
key-block tiles, globaltimer / clock64 at the tile's start and after its dK/dV epilogue.
Prints the effective clock, per-CTA cycles per query-tile step, the spread of CTA end times
and the per-tile fixed cost.   usage: python tools/tile_trace_bwd.py CAUSAL [N]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2307_08691_b200 as fa2

causal = len(sys.argv) > 1 and sys.argv[1] == "1"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
B, H, d = 16384 // N, 16, 128
q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = fa2.forward(q, k, v, causal=causal)
ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
run = lambda: fa2.backward(q, k, v, o, lse, do, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)
for _ in range(5):
    run()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
fl = 10.0 * N * N * d * H * B / (2 if causal else 1)
print(f"bwd causal={causal} N={N} B={B}: {ms * 1e3:.1f} us, {fl / ms / 1e9:.1f} TFLOP/s (untraced, whole backward)")
tr = torch.zeros(4096 + 148 * 32 * 8, dtype=torch.int64, device="cuda")
fa2.lib().fa2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
run()
fa2.lib().fa2_debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy()[4096:].reshape(148, 32, 8).astype(np.float64)
valid = t[:, :, 0] > 0
g0 = t[:, :, 0][valid].min()
dur_ns = np.where(valid, t[:, :, 2] - t[:, :, 0], np.nan)
dur_cy = np.where(valid, t[:, :, 3] - t[:, :, 1], np.nan)
nx = t[:, :, 5]
print(f"effective SM clock {np.nansum(dur_cy) / np.nansum(dur_ns):.3f} GHz; max tiles per CTA {valid.sum(1).max()}")
ends = np.nanmax(np.where(valid, t[:, :, 2] - g0, np.nan), axis=1) / 1e3
print(f"CTA end times (us): min {np.nanmin(ends):.1f} median {np.nanmedian(ends):.1f} max {np.nanmax(ends):.1f}")
cps = np.array([np.nansum(dur_cy[c]) / max(1, nx[c][valid[c]].sum()) for c in range(148)])
print("cycles per query-tile step per CTA: min %.0f p10 %.0f median %.0f p90 %.0f max %.0f" % (
    cps.min(), np.percentile(cps, 10), np.median(cps), np.percentile(cps, 90), cps.max()))
steps = np.array([nx[c][valid[c]].sum() for c in range(148)])
print("steps per CTA: min %d median %d max %d" % (steps.min(), np.median(steps), steps.max()))
m = valid
x, y = nx[m], dur_cy[m]
A = np.stack([np.ones_like(x), x], 1)
(a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"cycles = {a:.0f} + {b:.0f} * steps per tile (steps {x.min():.0f}-{x.max():.0f}); fixed share {a * len(x) / y.sum():.3f}")
gap = t[:, 1:, 0] - t[:, :-1, 2]
gm = valid[:, 1:] & valid[:, :-1]
print(f"inter-tile gap: mean {np.mean(gap[gm]) / 1e3:.2f} us")
ep = np.where(valid & (t[:, :, 7] > 0), t[:, :, 3] - t[:, :, 7], np.nan)
if np.isfinite(ep).any():
    print(f"epilogue (last MMAs' wait + dK/dV stores) cycles per tile: {np.nanmean(ep):.0f}")
