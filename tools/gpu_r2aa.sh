#!/bin/bash
# round 2: CTA-pair prefill, two softmax warps per sub-partition (fits 227 KiB now)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2aa
O=gpurun_out/r2aa
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VT_PREFILL_PAIR=1 timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_poisoned_tails_gpu.py -x -q > $O/pytest_pair.log 2>&1; echo "pytest pair rc=$?" >> $O/status
for v in 1 0 1 0; do
  VT_PREFILL_PAIR=$v timeout 300 python tools/kernel_bench.py --which prefill --iters 64 >> $O/pf_ab_$v.json 2>&1
done
VT_PREFILL_PAIR=1 VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf2trace.so timeout 300 python tools/trace_pair.py > $O/trace_pair.txt 2>&1; echo "trace rc=$?" >> $O/status
cat $O/status
