#!/usr/bin/env bash
# A/B of the cold 20k forward (Llama-3.1-8B) under env settings / library variants, alternating:
#   tools/ab_cold.sh "PREFILLONLY_LIB=build/variants/lib_prev.so" "X=1"
for rep in 1 2; do
  for cfg in "$@"; do
    echo "$cfg rep$rep $(env $cfg timeout 200 python tools/bench_engine.py 20000 2>&1 | grep '"tok_s"' | tail -1)"
  done
done
