#!/bin/bash
# round 2: QKV pair hand-off as 16-byte st.async into a padded feature-major buffer
cd "$(dirname "$0")/.."
O=gpurun_out/r2am; mkdir -p $O
timeout 600 python -m pytest tests/test_qkv_gpu.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/status
tail -2 $O/tests.log
for r in 1 2; do timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16,128,256 --qkv-split 0,2 2>>$O/kb.err | grep fused >> $O/kb.txt; done
bash tools/gpu_trace_qkv.sh > $O/trace.txt 2>&1
cat $O/status $O/kb.txt; grep -A30 "split=3" $O/trace.txt | grep -v "entry\|setup\|first_land"
