timeout 120 python tools/trace_bwd_pair.py
for r in 1 2; do timeout 300 python tools/kernel_ms.py; FA2_BWD_PAIR=1 timeout 300 python tools/kernel_ms.py; done
