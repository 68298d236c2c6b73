#!/bin/bash
# round 2: fused QKV split 3 (pair + L2 helper, 144 CTAs) vs split 2 (pair, 96 CTAs)
cd "$(dirname "$0")/.."
O=gpurun_out/r2af; mkdir -p $O
timeout 300 python -m pytest tests/test_qkv_gpu.py -x -q > $O/qkv_tests.log 2>&1; echo "tests rc=$?" >> $O/status
tail -3 $O/qkv_tests.log
for q8 in 2 1 3 2; do
  VT_QKV_HELPER_Q8=$q8 timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 2,3 2>>$O/kb.err | grep fused | sed "s/^/q8=$q8 /" >> $O/kb.txt
done
cat $O/status $O/kb.txt
