#!/usr/bin/env bash
# compute-sanitizer pass of the final tree (run under gpurun): memcheck (defaults, PO_SK=1) and synccheck over
# tools/sanitize.py's small invocations of every kernel path. Logs in gpurun_out/san2_*.log.
O=gpurun_out; mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py > $O/san2_mem_default.log 2>&1; echo "rc=$?" >> $O/san2_mem_default.log
PO_SK=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py > $O/san2_mem_sk1.log 2>&1; echo "rc=$?" >> $O/san2_mem_sk1.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize.py > $O/san2_sync.log 2>&1; echo "rc=$?" >> $O/san2_sync.log
