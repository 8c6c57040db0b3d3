./tools/micro/tmaio > gpurun_out/r2f_tmaio.txt 2>&1; cat gpurun_out/r2f_tmaio.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2f_pytest_gpu.log
python tools/kernel_ms.py
