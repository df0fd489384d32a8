O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/vl_gputests.log 2>&1; echo "tests rc=$?" >> $O/vl_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/vl_smoke.log 2>&1; echo "smoke rc=$?" >> $O/vl_smoke.log
timeout 900 python bench.py > $O/vl_bench.json 2> $O/vl_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/vl_bench_ref.json 2>&1
timeout 300 python tools/hit_classes.py > $O/vl_hit_classes.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/vl_hit_launches.csv python tools/hit_once.py 1 > /dev/null 2>&1
ls -la $O
