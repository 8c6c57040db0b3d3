timeout 120 python tools/pcie_bw.py
FA2_BWD_PAIR=0 timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_varlen_gpu.py -m gpu -x -q -k "backward or varlen or gqa" > gpurun_out/r2al_pytest.log 2>&1; echo "one-SM pytest $?"; tail -2 gpurun_out/r2al_pytest.log
for r in 1 2; do for v in cur5 cur6; do echo "== $v"; FA2_BWD_PAIR=0 FA2_LIB_PATH=variants/$v.so timeout 200 python tools/kernel_ms.py 2>&1 | tail -1; done; done
timeout 100 python tools/trace_bwd_pair.py
