#!/bin/bash
# round 2 (late): full GPU suite + smoke + default bench + reference arm, and an
# ncu --set full capture of the split-3 fused QKV kernel
cd "$(dirname "$0")/.."
O=gpurun_out/r2an; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qkv_append -s 6 -c 1 -o $O/qkv_split3 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 0 > $O/ncu_qkv.log 2>&1; echo "ncu rc=$?" >> $O/status
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status
timeout 300 python bench.py --impl reference > $O/benchref.json 2> $O/benchref.err; echo "ref rc=$?" >> $O/status
cat $O/status; tail -1 $O/pytest_gpu.log; tail -1 $O/smoke.log
