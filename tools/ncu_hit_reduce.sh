#!/bin/bash
# ncu --set full on the prefix-hit split-K reduce launches (QKV/RoPE, O and down residual), L2 left warm between
# kernels (--cache-control none) as inside a forward; run under gpurun, 1 GPU.
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:splitk_reduce \
  -c 8 -o $OUT/hit_reduce_full -f python tools/hit_once.py 1 > $OUT/ncu_hit_reduce.log 2>&1
ls -la $OUT/hit_reduce_full*
