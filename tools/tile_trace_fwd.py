"""Per-tile forward timeline (debug hook): for every CTA's first 16 work tiles and each
softmax warpgroup, globaltimer / clock64 at the tile's start and after its epilogue.
Prints the kernel span, the effective SM clock, the per-block period inside tiles, the
per-tile fixed cost (least squares: cycles = a + b * blocks) and the idle gaps.

usage: python tools/tile_trace_fwd.py D CAUSAL [N]"""
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
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    fa2.forward(q, k, v, causal=causal)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
fl = 4.0 * N * N * d * H * B / (2 if causal else 1)
print(f"d={d} causal={causal} N={N} B={B} H={H}: {ms * 1e3:.1f} us, {fl / ms / 1e9:.1f} TFLOP/s (untraced)")
tr = torch.zeros(65536, dtype=torch.int64, device="cuda")
fa2.lib().fa2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
fa2.forward(q, k, v, causal=causal)
fa2.lib().fa2_debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy()[4096:4096 + 148 * 16 * 2 * 8].reshape(148, 16, 2, 8)
valid = t[:, :, :, 0] > 0
g0 = t[:, :, :, 0][valid].min()
gs, cs, ge, ce = (t[:, :, :, i].astype(np.float64) for i in range(4))
nb = t[:, :, :, 5]
dur_ns = np.where(valid, ge - gs, np.nan)
dur_cy = np.where(valid, ce - cs, np.nan)
clk = np.nansum(dur_cy) / np.nansum(dur_ns)
span = (ge[valid].max() - g0) / 1e3
print(f"traced span {span:.1f} us, effective SM clock {clk:.3f} GHz, CTAs with tiles: {int(valid.any(axis=(1, 2)).sum())}")
# per CTA: busy time of wg 0 (sum of its tile durations) vs its span, and its end time
ends = np.nanmax(np.where(valid, ge - g0, np.nan), axis=(1, 2)) / 1e3
busy = np.nansum(np.where(valid[:, :, 0], dur_ns[:, :, 0], 0), axis=1) / 1e3
ok = ~np.isnan(ends)
print(f"CTA end times (us): min {np.nanmin(ends):.1f} median {np.nanmedian(ends):.1f} max {np.nanmax(ends):.1f}; "
      f"wg0 busy / end (median) {np.median(busy[ok] / ends[ok]):.3f}")
for w in (0, 1):
    m = valid[:, :, w] & (nb[:, :, w] > 0)
    x, y = nb[:, :, w][m].astype(np.float64), dur_cy[:, :, w][m]
    A = np.stack([np.ones_like(x), x], 1)
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    print(f"wg{w}: {m.sum()} tiles, blocks/tile {x.min():.0f}-{x.max():.0f} (mean {x.mean():.1f}); "
          f"cycles = {a:.0f} + {b:.0f} * blocks; fixed share {a * len(x) / y.sum():.3f}")
# gaps between consecutive tiles of the same warpgroup (end of n -> start of n+1)
gap = (gs[:, 1:, 0] - ge[:, :-1, 0])
gm = valid[:, 1:, 0] & valid[:, :-1, 0]
print(f"wg0 inter-tile gap: mean {np.mean(gap[gm]) / 1e3:.2f} us, total per CTA {np.sum(np.where(gm, gap, 0), axis=1).mean() / 1e3:.1f} us")
first = (gs[:, 0, 0] - g0)[valid[:, 0, 0]] / 1e3
print(f"first tile start after kernel's first: mean {first.mean():.2f} us max {first.max():.2f} us")
# per-CTA speed: cycles per key block over its tiles (wg 0), against its SM id and tile count
smid = t[:, 0, 0, 6]
cpb = np.array([np.nansum(dur_cy[c, :, 0]) / max(1, nb[c, :, 0][valid[c, :, 0]].sum()) for c in range(148)])
ntl = valid[:, :, 0].sum(axis=1)
o = np.argsort(cpb)
print("cycles/block per CTA: min %.0f p10 %.0f median %.0f p90 %.0f max %.0f" % (
    cpb[o[0]], np.percentile(cpb, 10), np.median(cpb), np.percentile(cpb, 90), cpb[o[-1]]))
print("slowest 10 CTAs (cta, smid, tiles, cyc/blk, end us):",
      [(int(c), int(smid[c]), int(ntl[c]), round(float(cpb[c])), round(float(ends[c]), 1)) for c in o[-10:]])
print("fastest 5 CTAs:", [(int(c), int(smid[c]), int(ntl[c]), round(float(cpb[c])), round(float(ends[c]), 1)) for c in o[:5]])
# by SM id parity / TPC (smid // 2) -- is the slowness tied to the SM's position?
by_tpc = {}
for c in range(148):
    by_tpc.setdefault(int(smid[c]) // 2, []).append(cpb[c])
print("cyc/blk by smid//16 (GPC-ish):", [round(float(np.mean([cpb[c] for c in range(148) if smid[c] // 16 == gg])))
                                        for gg in range(10) if any(smid[c] // 16 == gg for c in range(148))])
# pair kernel: clock64 at the epilogue's start (slot 7) -> tile end: epilogue cycles per tile
ep = np.where(valid & (t[:, :, :, 7] > 0), t[:, :, :, 3].astype(np.float64) - t[:, :, :, 7], np.nan)
if np.isfinite(ep).any():
    print("epilogue (last P~V wait + O/L stores) cycles per tile: wg0 %.0f wg1 %.0f" % (np.nanmean(ep[:, :, 0]), np.nanmean(ep[:, :, 1])))
