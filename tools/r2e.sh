for r in 1 2; do
for v in base pair_noex pair_nored pair_both; do
  echo "== $v round $r"; FA2_BWD_PAIR=1 FA2_LIB_PATH=variants/$v.so timeout 300 python tools/kernel_ms.py 2>&1 | tail -1
done; done > gpurun_out/r2e_ab.txt 2>&1
for v in pair_noex pair_nored pair_both; do
  echo "== $v trace"; FA2_BWD_PAIR=1 FA2_LIB_PATH=variants/$v.so timeout 120 python tools/trace_bwd128.py 2>&1 | tail -7
done > gpurun_out/r2e_trace.txt 2>&1
cat gpurun_out/r2e_ab.txt gpurun_out/r2e_trace.txt
