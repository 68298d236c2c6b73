#!/bin/bash
# round 2: fused QKV — token-split multicast pair (VT_QKV_MODE=mc) vs the K-split pair
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2s
O=gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VT_QKV_MODE=mc timeout 600 python -m pytest tests/test_qkv_gpu.py -x -q > $O/pytest_mc.log 2>&1; echo "pytest mc rc=$?" >> $O/status
for rep in 1 2; do
  timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,128,256 >> $O/qkv_ksplit.json 2>&1
  VT_QKV_MODE=mc timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,128,256 >> $O/qkv_mc.json 2>&1
done
VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkvtrace.so timeout 300 python tools/trace_qkv.py 64 0 > $O/trace_ksplit.txt 2>&1
VT_QKV_MODE=mc VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkvtrace.so timeout 300 python tools/trace_qkv.py 64 0 > $O/trace_mc.txt 2>&1
echo "trace rc=$?" >> $O/status
cat $O/status
