#!/usr/bin/env bash
# A/B the attention variants built by tools/build_variant.sh: parity (test_gpu_attention) + timing per variant.
#   tools/ab_attn.sh base v1 v2 ...     (base = the in-tree library)
for v in "$@"; do
  lib=paper_2505_07203_b200/libprefillonly.so
  [ "$v" != base ] && lib=build/variants/lib_$v.so
  echo "== $v"
  PREFILLONLY_LIB=$lib timeout 120 python -m pytest -q -x tests/test_gpu_attention.py 2>&1 | tail -1
  PREFILLONLY_LIB=$lib timeout 90 python tools/bench_attn.py 2>&1 | tail -4
done
