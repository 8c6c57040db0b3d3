"""Time forward/backward of one or more library builds (FA2_LIB_PATH) on paper shapes."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import json, math, sys, torch
import paper_2307_08691_b200 as fa2
sys.stderr.write(fa2.__file__ + "\n")
res = {}
for (d, H) in ((128, 16), (64, 32)):
    for causal in (False, True):
        N = 8192; B = 2
        q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
        o, lse = fa2.forward(q, k, v, causal=causal)
        ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        def tm(fn, reps=20):
            for _ in range(3): fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps): fn()
            e.record(); torch.cuda.synchronize()
            return s.elapsed_time(e) / reps
        fl = 4.0 * N * N * d * H * B / (2 if causal else 1)
        tf = tm(lambda: fa2.forward(q, k, v, causal=causal, out=o, lse=lse))
        tb = tm(lambda: fa2.backward(q, k, v, o, lse, do, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)) if "bwd" in sys.argv else float("nan")
        # accuracy vs fp32 torch reference on one head
        qf, kf, vf = (t[0, 0].float() for t in (q, k, v))
        s_ = (qf @ kf.T) / math.sqrt(d)
        if causal: s_ = s_.masked_fill(torch.triu(torch.ones(N, N, device="cuda", dtype=torch.bool), 1), float("-inf"))
        ref = torch.softmax(s_, -1) @ vf
        err = (o[0, 0].float() - ref).abs().max().item()
        res[f"d{d}_c{int(causal)}"] = {"fwd_tflops": round(fl / tf / 1e9, 1), "bwd_tflops": round(2.5 * fl / tb / 1e9, 1), "o_err": err}
print(json.dumps(res))
'''

if __name__ == "__main__":
    out = {}
    for lib in sys.argv[1:]:
        if lib == "bwd":
            continue
        if os.path.isdir(lib):   # a checkout: use its own binding and library (A/B across API changes)
            env = dict(os.environ, PYTHONPATH=os.path.abspath(lib))
            env.pop("FA2_LIB_PATH", None)
        else:
            env = dict(os.environ, FA2_LIB_PATH=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CHILD] + (["bwd"] if "bwd" in sys.argv else []), env=env,
                           cwd=os.path.abspath(lib) if os.path.isdir(lib) else None, capture_output=True, text=True,
                           timeout=600)
        out[os.path.basename(lib)] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
        print(os.path.basename(lib), out[os.path.basename(lib)], flush=True)
