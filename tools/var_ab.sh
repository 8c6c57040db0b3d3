# A/B timing of library variants (variants/*.so, built off-tree) on one box.
# usage: tools/var_ab.sh TAG "v1 v2 ..." [reps]
TAG=$1; VARS=$2; REPS=${3:-2}
for r in $(seq $REPS); do
for v in $VARS; do
  echo "== $v round $r"
  FA2_LIB_PATH=variants/$v.so timeout 300 python tools/kernel_ms.py 2>&1 | tail -1
done; done > gpurun_out/${TAG}_ab.txt 2>&1
for v in $VARS; do
  echo "== $v trace"; FA2_LIB_PATH=variants/$v.so timeout 120 python tools/trace_bwd128.py 2>&1 | tail -7
done > gpurun_out/${TAG}_trace.txt 2>&1
cat gpurun_out/${TAG}_ab.txt gpurun_out/${TAG}_trace.txt
