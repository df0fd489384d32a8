#!/bin/bash
# Does the MLP intermediate (gate/up output -> down input) reach HBM? DRAM bytes per launch with L2 state kept across
# kernels (--cache-control none) for chunk = 8192 (default) and chunk = 2048 (the 58.7 MB act buffer fits L2).
OUT=gpurun_out; mkdir -p $OUT
for ch in 8192 2048; do
  timeout 900 ncu --cache-control none --clock-control none -k regex:gemm2_kernel -s 200 -c 24 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $OUT/mlp_l2_$ch.csv \
    python tools/bench_engine.py 20000 $ch > /dev/null 2>&1
done
ls -la $OUT/mlp_l2_*.csv
