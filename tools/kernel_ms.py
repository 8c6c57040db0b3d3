"""Per-kernel device times (fwd, bwd preprocess, bwd main, dQ convert) through the
library's timing hook, for the paper shapes; run from a checkout root (cwd) so that
checkout's binding and library are used."""
import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2307_08691_b200 as fa2

out = {}
for (d, H) in ((128, 16), (64, 32)):
    for causal in (False, True):
        B, N = 2, 8192
        q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
        o, lse = fa2.forward(q, k, v, causal=causal)
        ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        for e in ev:   # torch creates the CUDA event lazily, on its first record
            e.record()
        torch.cuda.synchronize()
        keep = fa2.set_timing_events(ev)
        acc = [0.0] * 5
        reps = 10
        for it in range(3 + reps):
            fa2.forward(q, k, v, causal=causal, out=o, lse=lse)
            fa2.backward(q, k, v, o, lse, do, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)
            torch.cuda.synchronize()
            if it >= 3:
                for j in range(5):
                    acc[j] += ev[j].elapsed_time(ev[j + 1]) / reps
        fa2.set_timing_events(None)
        out[f"d{d}_c{int(causal)}"] = {n: round(x * 1000, 1) for n, x in zip(("fwd", "gap", "pre", "main", "dq"), acc)}
print(json.dumps(out))
