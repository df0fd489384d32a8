#!/usr/bin/env bash
# In-kernel split-KV combine A/B (run under gpurun): attention + engine tests, then the warm prefix-hit forward with
# the separate combine launch (PO_ATTN_COMBINE=0) and the in-kernel combine (PO_ATTN_COMBINE=1).
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_engine.py tests/test_gpu_parity_fullsize.py -q -x -p no:cacheprovider > $O/c_tests.log 2>&1; echo "tests rc=$?" >> $O/c_tests.log
timeout 600 python tools/hit_ab.py 'PO_ATTN_COMBINE=0' 'PO_ATTN_COMBINE=1' > $O/c_hit_ab.log 2>&1
