timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2x_pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-tables --no-e2e --extras --steps 5 > gpurun_out/r2x_extras.json 2> gpurun_out/r2x_extras.err; echo "extras $?"
python3 -c "
import json; j=json.loads(open('gpurun_out/r2x_extras.json').read().strip().splitlines()[-1])
for r in j['extras']: print(r)
"
