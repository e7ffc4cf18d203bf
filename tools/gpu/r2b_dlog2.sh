for v in anch4 anch16; do echo "== $v"; GLA_LIB=$PWD/variants/libgla_$v.so timeout 1200 python tools/dlog_err.py 2>&1 | grep saved; done
