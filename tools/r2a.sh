set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name())"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2a_pytest_gpu.log
FA2_BWD_PAIR=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -m gpu -x -q -k "backward or bwd or full" > gpurun_out/r2a_pytest_pair.log 2>&1; echo "pair pytest exit $?"; tail -3 gpurun_out/r2a_pytest_pair.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench exit $?"; cat gpurun_out/r2a_bench.json | head -c 2500
for i in 1 2; do
timeout 300 python tools/kernel_ms.py > gpurun_out/r2a_kms_single$i.json; cat gpurun_out/r2a_kms_single$i.json
FA2_BWD_PAIR=1 timeout 300 python tools/kernel_ms.py > gpurun_out/r2a_kms_pair$i.json; cat gpurun_out/r2a_kms_pair$i.json
done
