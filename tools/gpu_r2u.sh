#!/bin/bash
# round 2: fused QKV — weights issued at barrier init, partial into its own buffer (no handshake)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2u
O=gpurun_out/r2u
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_qkv_gpu.py -x -q > $O/pytest_qkv.log 2>&1; echo "pytest qkv rc=$?" >> $O/status
for rep in 1 2; do
  timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,128,256 >> $O/qkv_new.json 2>&1
  VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkvold.so timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,128,256 >> $O/qkv_old.json 2>&1
done
VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkvtrace.so timeout 300 python tools/trace_qkv.py 64 0 > $O/trace_new.txt 2>&1
echo "trace rc=$?" >> $O/status
cat $O/status
