#!/bin/bash
# ncu --set full on the prefix-hit path's kernels (run under gpurun, 1 GPU): the packed short-query attention and the
# short-M QKV / gate-up GEMMs of one warm hit forward (tools/hit_once.py 1: launches after the cold forward).
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 40 -c 1 -o $OUT/hit_attn_full -f \
  python tools/hit_once.py 1 > $OUT/ncu_hit_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 300 -c 4 -o $OUT/hit_gemm_full -f \
  python tools/hit_once.py 1 > $OUT/ncu_hit_gemm.log 2>&1
ls -la $OUT/hit_*full*
