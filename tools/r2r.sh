timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fp8_gpu.py tests/test_varlen_gpu.py -m gpu -x -q -k "forward or fp8 or varlen or rectangular" > gpurun_out/r2r_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/r2r_pytest.log
for r in 1 2 3; do for v in cur tmax; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 300 python tools/fwd_ms.py 2>&1 | tail -1; done; done
