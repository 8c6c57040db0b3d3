set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > gpurun_out/r2f_ncu_bench.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa2_bwd_pair -s 3 -c 1 -o gpurun_out/r2f_prof_bwd \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > gpurun_out/r2f_ncu_bwd.log 2>&1; echo "ncu bwd $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa2_fwd_pair -s 3 -c 1 -o gpurun_out/r2f_prof_fwd \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > gpurun_out/r2f_ncu_fwd.log 2>&1; echo "ncu fwd $?"
timeout 600 ncu --set full --clock-control none -k regex:fa2_bwd_preprocess -s 3 -c 1 -o gpurun_out/r2f_prof_pre \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > gpurun_out/r2f_ncu_pre.log 2>&1; echo "ncu pre $?"
timeout 600 ncu --set full --clock-control none -k regex:fa2_dq_convert -s 3 -c 1 -o gpurun_out/r2f_prof_dq \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > gpurun_out/r2f_ncu_dq.log 2>&1; echo "ncu dq $?"
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/r2f_memcheck.log 2>&1; echo "memcheck $?"; tail -2 gpurun_out/r2f_memcheck.log
