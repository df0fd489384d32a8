#!/usr/bin/env bash
# One GPU evidence pass (run under gpurun): tests, smoke, both bench arms, launch lists of a cold step and of a
# prefix-hit forward. Outputs in gpurun_out/; summaries are copied into profiles/ by hand.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/ev_gputests.log 2>&1; echo "tests rc=$?" >> $O/ev_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/ev_smoke.log 2>&1
timeout 900 python bench.py > $O/ev_bench.json 2> $O/ev_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/ev_bench_ref.json 2>&1
timeout 300 python tools/hit_once.py > $O/ev_hit.log 2>&1
PO_STREAM=1 timeout 300 python tools/hit_once.py > $O/ev_hit_stream.log 2>&1
timeout 300 python tools/bench_stream.py > $O/ev_bench_stream.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/ev_hit_launches.csv python tools/hit_once.py 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 460 --csv --log-file $O/ev_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-qps --no-cpu-baseline > /dev/null 2>&1
ls -la $O
