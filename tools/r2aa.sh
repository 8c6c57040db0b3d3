for v in det1 det0; do echo "== $v"; FA2_LIB_PATH=variants/$v.so timeout 60 python tools/det_debug.py; done
