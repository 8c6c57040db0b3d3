timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2g_pytest_gpu.log
for r in 1 2; do for v in base fwd_rel fwd_relacq; do echo "== $v"; FA2_LIB_PATH=variants/$v.so python tools/fwd_ms.py 2>&1 | tail -2; done; done
