#!/bin/bash
# round 2: fused QKV with a 96 KiB ring (two CTAs per SM: the next launch's
# weight ring fills while this one reduces) vs the 192 KiB ring
cd "$(dirname "$0")/.."
O=gpurun_out/r2ac; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for small in 0 1 0 1; do
  VT_QKV_RING_SMALL=$small timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 >> $O/kb_small$small.jsonl 2>>$O/kb.err
done
VT_QKV_RING_SMALL=1 timeout 300 python -m pytest tests/test_qkv_gpu.py -x -q > $O/qkv_tests_small.log 2>&1; echo "tests small rc=$?" >> $O/status
VT_QKV_RING_SMALL=1 timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 16,32 >> $O/kb_small1_b.jsonl 2>>$O/kb.err
VT_QKV_RING_SMALL=0 timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 16,32 >> $O/kb_small0_b.jsonl 2>>$O/kb.err
cat $O/status; grep fused $O/kb_small*.jsonl
timeout 600 python tools/prefill_vs_libs.py > $O/prefill_vs_libs.jsonl 2> $O/prefill_vs_libs.err; echo "pvl rc=$?" >> $O/status; cat $O/prefill_vs_libs.jsonl; tail -3 $O/prefill_vs_libs.err
