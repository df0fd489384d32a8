#!/usr/bin/env bash
# Split-K reduce A/B (run under gpurun): GEMM + engine tests on the built library, then the warm prefix-hit forward on
# build/variants/lib_old.so (previous reduce kernel) vs the in-tree library, and ncu of the reduce launches.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py tests/test_gpu_engine.py tests/test_gpu_parity_fullsize.py -q -x -p no:cacheprovider > $O/r_tests.log 2>&1; echo "tests rc=$?" >> $O/r_tests.log
timeout 900 python tools/hit_ab.py 'PREFILLONLY_LIB=build/variants/lib_old.so' 'PREFILLONLY_LIB=paper_2505_07203_b200/libprefillonly.so' > $O/r_hit_ab.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none -k regex:"splitk_reduce|attn_combine" \
  -c 12 -o $O/hit_reduce_i32 -f python tools/hit_once.py 1 > $O/ncu_red.log 2>&1
