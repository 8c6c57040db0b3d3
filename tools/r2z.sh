for r in 1 2; do for v in cur3 d64emu0 d64emu8 d64emu10 d64emu12; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 200 python tools/fwd_ms.py 2>&1 | tail -1; done; done
for v in cur3 d64emu0 d64emu12; do echo "== $v trace"; FA2_LIB_PATH=variants/$v.so timeout 100 python tools/trace_fwd.py 64 0 | tail -5; done
