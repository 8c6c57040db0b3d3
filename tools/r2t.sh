timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_varlen_gpu.py tests/test_parity_full_gpu.py -m gpu -x -q -k "forward or varlen or rectangular or PS64" > gpurun_out/r2t_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/r2t_pytest.log
timeout 100 python tools/trace_fwd.py 64 0 | tail -5
for r in 1 2; do for v in cur2 defer; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 300 python tools/fwd_ms.py 2>&1 | tail -1; done; done
