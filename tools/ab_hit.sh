#!/usr/bin/env bash
# A/B of prefix-hit forward service time under env settings: tools/ab_hit.sh "PO_SKINNY=0" "PO_SKINNY=1" ...
for cfg in "$@"; do
  for rep in 1 2 3; do
    echo "$cfg rep$rep $(env $cfg timeout 120 python tools/hit_once.py 2>&1 | tail -1)"
  done
done
