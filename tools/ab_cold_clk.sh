#!/usr/bin/env bash
# tools/ab_cold.sh with the SM clock and board power sampled (50 ms) during each run: median MHz / W under load
for rep in 1 2; do
  for cfg in "$@"; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 50 > /tmp/clk.csv &
    smi=$!
    line=$(env $cfg timeout 200 python tools/bench_engine.py 20000 2>&1 | grep '"tok_s"' | tail -1)
    kill $smi; wait $smi 2>/dev/null
    clk=$(python -c "
import statistics as s
r=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
r=[(float(a),float(b)) for a,b in r if float(b)>600]
print('MHz', s.median(a for a,_ in r) if r else 0, 'W', s.median(b for _,b in r) if r else 0, 'n', len(r))")
    echo "$cfg rep$rep $line $clk"
  done
done
