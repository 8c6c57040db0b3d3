timeout 400 python -m pytest tests/test_deterministic_gpu.py -m gpu -x -q > gpurun_out/r2y_det.log 2>&1; echo "det exit $?"; tail -5 gpurun_out/r2y_det.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2y_pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline --no-tables --no-e2e --no-check --extras --steps 5 > gpurun_out/r2y_extras.json 2> gpurun_out/r2y_extras.err; echo "extras $?"
python3 -c "
import json; j=json.loads(open('gpurun_out/r2y_extras.json').read().strip().splitlines()[-1])
for r in j['extras']: print(r)
"
