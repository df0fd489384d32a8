for v in 1_4 3_8 1_2 5_8 3_4; do echo "variant $v"; PREFILLONLY_LIB=build/variants/lib_$v.so timeout 120 python tools/bench_attn.py 2>&1 | head -2; done
