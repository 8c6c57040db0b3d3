timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2w_pytest_gpu.log
for r in 1 2; do for v in cur2 cpair; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 300 python tools/fwd_ms.py 2>&1 | tail -1; done; done
