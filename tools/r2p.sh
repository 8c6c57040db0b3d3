timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2p_pytest_gpu.log
bash tools/var_ab.sh r2p "cur emu2 emu6 emu8" 2 > /dev/null 2>&1; cat gpurun_out/r2p_ab.txt | python3 -c "
import sys,json
cur=None
for l in sys.stdin:
    if l.startswith('=='): cur=l.strip()
    elif l.startswith('{'):
        j=json.loads(l); print(cur, j['d128_c0']['main'], j['d128_c1']['main'])
"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "bench $?"
