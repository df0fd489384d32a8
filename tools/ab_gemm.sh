echo "== pair (2-CTA)"; timeout 200 python tools/bench_gemm.py
echo "== 1-CTA"; PO_GEMM_1CTA=1 timeout 200 python tools/bench_gemm.py
