for n in "$@"; do echo "== $n"; FA2_LIB_PATH=variants/lib_$n.so timeout 60 python tools/trace_fwd.py 128 2>&1 | tail -7; done
