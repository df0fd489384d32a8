for i in 1 2; do
echo "new"; timeout 120 python tools/bench_attn.py 2>&1 | head -2
echo "prev"; PREFILLONLY_LIB=build/ab/lib_prev.so timeout 120 python tools/bench_attn.py 2>&1 | head -2
done
