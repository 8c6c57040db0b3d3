timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_varlen_gpu.py tests/test_parity_full_gpu.py -m gpu -x -q -k "forward or varlen or rectangular or PS64" > gpurun_out/r2ag_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/r2ag_pytest.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-check --sweep --extras --steps 10 > gpurun_out/r2ag_sweep.json 2> gpurun_out/r2ag_sweep.err; echo "sweep $?"
python3 -c "
import json; j=json.loads(open('gpurun_out/r2ag_sweep.json').read().strip().splitlines()[-1])
for r in j['sweep']: print(r)
for r in j['extras']: print(r)
"
