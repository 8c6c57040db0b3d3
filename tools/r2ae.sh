timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2ae_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2ae_pytest_gpu.log
timeout 300 python tools/bench_det.py
timeout 600 python bench.py > gpurun_out/r2ae_bench.json 2> gpurun_out/r2ae_bench.err; echo "bench $?"
python3 -c "
import json; j=json.loads(open('gpurun_out/r2ae_bench.json').read().strip().splitlines()[-1])
print(j['value'], j['passes'], j['clocks'], j['roofline']['achieved'], j['roofline']['frac'], j['roofline']['kernel_ms'], j['shard_check']['fwd_bitwise'], j['shard_check']['bwd_deterministic_bitwise'])
"
