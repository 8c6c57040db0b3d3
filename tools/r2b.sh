set -x
python tools/trace_bwd128.py > gpurun_out/r2b_trace_single.txt 2>&1
FA2_BWD_PAIR=1 python tools/trace_bwd128.py > gpurun_out/r2b_trace_pair.txt 2>&1
cat gpurun_out/r2b_trace_single.txt gpurun_out/r2b_trace_pair.txt
FA2_BWD_PAIR=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa2_bwd_pair -s 2 -c 1 -o gpurun_out/r2b_prof_bwdpair python tools/bwd_once.py > gpurun_out/r2b_ncu1.log 2>&1; echo "ncu pair $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa2_bwd128 -s 2 -c 1 -o gpurun_out/r2b_prof_bwd1 python tools/bwd_once.py > gpurun_out/r2b_ncu2.log 2>&1; echo "ncu single $?"
