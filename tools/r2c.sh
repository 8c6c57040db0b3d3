set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "binding or launch" > gpurun_out/r2c_pytest.log 2>&1; tail -3 gpurun_out/r2c_pytest.log
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench $?"; tail -3 gpurun_out/r2c_bench.err
timeout 600 python bench.py --config gpt --steps 10 --no-cpu-baseline --no-tables > gpurun_out/r2c_gpt.json 2> gpurun_out/r2c_gpt.err; echo "gpt $?"; tail -3 gpurun_out/r2c_gpt.err
for n in 16384 32768 65536; do
timeout 600 python bench.py --config lc --seqlen $n --steps 5 --no-cpu-baseline --no-tables --no-e2e > gpurun_out/r2c_lc$n.json 2> gpurun_out/r2c_lc$n.err; echo "lc $n $?"; tail -3 gpurun_out/r2c_lc$n.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c_ref.json; echo "ref $?"
