timeout 400 python -m pytest tests/test_parity_gpu.py tests/test_varlen_gpu.py tests/test_deterministic_gpu.py -m gpu -x -q -k "gqa or backward or determ or varlen" > gpurun_out/r2an_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/r2an_pytest.log
cat > /tmp/mqa.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2307_08691_b200 as fa2
def tm(fn, reps=10):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for hkv in (1, 2, 8):
    for causal in (False, True):
        B, H, N, d = 2, 32, 8192, 128
        q, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(2))
        k, v = (torch.randn(B, hkv, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(2))
        o, lse = fa2.forward(q, k, v, causal=causal)
        ws = torch.empty(fa2.backward_workspace_size(B, H, N, d), dtype=torch.uint8, device="cuda")
        t = tm(lambda: fa2.backward(q, k, v, o, lse, do, causal=causal, workspace=ws))
        fl = 2.5 * 4.0 * N * N * d * H * B / (2 if causal else 1)
        print(f"H_kv={hkv} causal={causal}: bwd {fl / t / 1e9:.1f} TFLOP/s", flush=True)
PY
for v in cur6 hsplit; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 200 python /tmp/mqa.py; done
