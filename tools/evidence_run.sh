#!/usr/bin/env bash
# One GPU evidence pass (run under gpurun): tests, smoke, both bench arms, launch lists of a cold step and of a
# prefix-hit forward, ncu --set full of the dominant kernel (gate/up) and of attention. Outputs in gpurun_out/ev_*;
# summaries are copied into profiles/ by hand (see profiles/INDEX.md).
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/ev_gputests.log 2>&1; echo "tests rc=$?" >> $O/ev_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/ev_smoke.log 2>&1
timeout 900 python bench.py > $O/ev_bench.json 2> $O/ev_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/ev_bench_ref.json 2>&1
timeout 300 python tools/hit_once.py > $O/ev_hit.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/ev_hit_launches.csv python tools/hit_once.py 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 460 \
  --csv --log-file $O/ev_launches.csv python bench.py --steps 1 --warmup 3 --no-qps --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 71 -c 1 -o $O/ev_gemm_gateup_full -f \
  python tools/bench_gemm.py > $O/ev_ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 7 -c 1 -o $O/ev_attn_full -f \
  python tools/bench_attn.py > $O/ev_ncu_attn.log 2>&1
timeout 300 python tools/attn_vs_libs.py > $O/ev_attn_vs_libs.jsonl 2>&1
timeout 300 python tools/bench_gemm.py > $O/ev_gemm_vs_cublas.jsonl 2>&1
timeout 300 python tools/hit_classes.py > $O/ev_hit_classes.txt 2>&1
timeout 600 python tools/bench_configs.py llama128k $O/ev_config_llama128k.json > $O/ev_128k.log 2>&1
ls -la $O
