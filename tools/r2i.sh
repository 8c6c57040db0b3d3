timeout 120 ./tools/micro/dsmemcp
FA2_BWD_PAIR=1 timeout 120 python tools/trace_bwd_pair.py
