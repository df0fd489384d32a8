#!/bin/bash
# ncu evidence (run under gpurun, 1 GPU). Outputs land in gpurun_out/; tools/ncu_summary.py writes profiles/.
OUT=gpurun_out
mkdir -p $OUT
# 1) launch list of one bench step (cold-cache serialised per-launch times: compare SHARES)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 460 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-qps --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
# 2) full set on the attention kernel at 20k tokens (first 20k launch of tools/bench_attn.py: skip 7 4k launches)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 7 -c 1 -o $OUT/attn_full -f \
  python tools/bench_attn.py > $OUT/ncu_attn.log 2>&1
# 3) full set on the fused gate/up GEMM (EPI_SILU_MUL, 8192x28672x4096: pair-kernel launches 69..91 of bench_gemm)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 71 -c 1 -o $OUT/gemm_gateup_full -f \
  python tools/bench_gemm.py > $OUT/ncu_gemm.log 2>&1
# 4) full set on the down GEMM with the residual epilogue (8192x4096x14336: launches 92..114)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 94 -c 1 -o $OUT/gemm_down_full -f \
  python tools/bench_gemm.py > $OUT/ncu_gemm2.log 2>&1
ls -la $OUT
