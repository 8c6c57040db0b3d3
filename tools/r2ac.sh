timeout 400 python -m pytest tests/test_deterministic_gpu.py -m gpu -x -q > gpurun_out/r2ac_det.log 2>&1; echo "det exit $?"; tail -3 gpurun_out/r2ac_det.log
timeout 200 python tools/bench_det.py > gpurun_out/r2ac_bench_det.txt 2>&1; echo "bench_det $?"; tail -12 gpurun_out/r2ac_bench_det.txt
