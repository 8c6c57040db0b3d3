#!/bin/bash
# One gpurun session: GPU tests, bench, ncu launch list and full profiles.
# usage: tools/gpu_round.sh TAG [tests|bench|ncu|all]
TAG=${1:-r}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/${TAG}_pytest_gpu.log
  tail -5 $OUT/${TAG}_pytest_gpu.log
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit $?"
  cat $OUT/${TAG}_bench.json | head -c 3000; echo
  tail -3 $OUT/${TAG}_bench.err
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > $OUT/${TAG}_ncu_bench.log 2>&1; echo "ncu launches exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fa2_bwd.*kernel" -s 3 -c 1 -o $OUT/${TAG}_prof_bwd \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > $OUT/${TAG}_ncu_bwd.log 2>&1; echo "ncu bwd exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa2_fwd -s 3 -c 1 -o $OUT/${TAG}_prof_fwd \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tables --no-check > $OUT/${TAG}_ncu_fwd.log 2>&1; echo "ncu fwd exit $?"
fi
