#!/bin/bash
# round 2: split 3 with a feature-major helper partial (16-byte stores/loads, one release); helper share sweep
cd "$(dirname "$0")/.."
O=gpurun_out/r2aj; mkdir -p $O
timeout 300 python -m pytest tests/test_qkv_gpu.py -x -q > $O/qkv_tests.log 2>&1; echo "tests rc=$?" >> $O/status
tail -2 $O/qkv_tests.log
for q in 16 20 16 20; do
  VT_QKV_HELPER_Q64=$q timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 2,3 2>>$O/kb.err | grep '"fused\|(fused' | sed "s/^/q64=$q /" >> $O/kb.txt
done
cat $O/status $O/kb.txt
bash tools/gpu_trace_qkv.sh > $O/trace.txt 2>&1; grep -A30 "split=3" $O/trace.txt
