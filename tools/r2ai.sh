for r in 1 2 3; do for v in cur5 pe1 pe3 pe3s pe4s; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 200 python tools/fwd_ms.py 2>&1 | tail -1; done; done
