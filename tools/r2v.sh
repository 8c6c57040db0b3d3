timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2v_pytest_gpu.log
timeout 300 python tools/kernel_ms.py
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench $?"
python3 -c "
import json; j=json.loads(open('gpurun_out/r2v_bench.json').read().strip().splitlines()[-1])
print(j['value'], j['passes'], j['clocks'], j['roofline']['kernel_ms'])
for r in j['short_n']: print(r)
"
