FA2_BWD_PAIR=1 timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "backward and 128" > gpurun_out/r2j_pair_small.log 2>&1; echo "small $?"; tail -15 gpurun_out/r2j_pair_small.log
FA2_BWD_PAIR=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -m gpu -x -q -k "backward or bwd or full or gqa" > gpurun_out/r2j_pair.log 2>&1; echo "pair pytest $?"; tail -3 gpurun_out/r2j_pair.log
for r in 1 2; do
timeout 300 python tools/kernel_ms.py; FA2_BWD_PAIR=1 timeout 300 python tools/kernel_ms.py
done
FA2_BWD_PAIR=1 timeout 120 python tools/trace_bwd_pair.py
