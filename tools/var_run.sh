#!/bin/bash
# Run fwd trace + fwd_ms for each variant library under variants/ (A/B experiments).
# usage: tools/var_run.sh TAG name1 name2 ...
TAG=$1; shift
mkdir -p gpurun_out
for n in "$@"; do
  echo "== $n" >> gpurun_out/${TAG}_var.txt
  FA2_LIB_PATH=variants/lib_$n.so timeout 60 python tools/trace_fwd.py 128 2>&1 | tail -12 >> gpurun_out/${TAG}_var.txt
  FA2_LIB_PATH=variants/lib_$n.so timeout 90 python tools/fwd_ms.py 2>&1 | tail -2 >> gpurun_out/${TAG}_var.txt
done
cat gpurun_out/${TAG}_var.txt
