O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/v_gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/v_gputests.log 2>&1; echo "tests rc=$?" >> $O/v_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/v_smoke.log 2>&1; echo "smoke rc=$?" >> $O/v_smoke.log
timeout 900 python bench.py > $O/v_bench.json 2> $O/v_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/v_bench_ref.json 2>&1
timeout 300 python tools/hit_classes.py > $O/v_hit_classes.txt 2>&1
ls -la $O
