#!/bin/bash
# ncu --set full of one warm prefix-hit forward's kernels on the final tree (run under gpurun, 1 GPU), L2 left warm
# between kernels as inside a forward: split-K swap GEMMs, stream-K gate/up, split-K reduce, split-KV combine, attention.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
  -k regex:'gemm2s_kernel|gemm_sk_kernel|splitk_reduce|attn_combine' -s 2 -c 8 -o $OUT/hitfin_gemm_full -f \
  python tools/hit_once.py 1 > $OUT/ncu_hitfin_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:attn_fwd -s 33 -c 1 \
  -o $OUT/hitfin_attn_full -f python tools/hit_once.py 1 > $OUT/ncu_hitfin_attn.log 2>&1
ls -la $OUT/hitfin_*
