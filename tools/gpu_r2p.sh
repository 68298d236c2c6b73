#!/bin/bash
# round 2: CTA-pair prefill with two softmax warps per sub-partition (one per
# 128-column half): parity, A/B against the single-CTA kernel, timelines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2p
O=gpurun_out/r2p
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VT_PREFILL_PAIR=1 timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_poisoned_tails_gpu.py -x -q > $O/pytest_pair.log 2>&1; echo "pytest pair rc=$?" >> $O/status
VT_PREFILL_PAIR=1 VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf2nreg.so timeout 600 python -m pytest tests/test_prefill_gpu.py -x -q > $O/pytest_pair_nreg.log 2>&1; echo "pytest pair nreg rc=$?" >> $O/status
for v in 1 0 1 0; do
  VT_PREFILL_PAIR=$v timeout 300 python tools/kernel_bench.py --which prefill --iters 64 >> $O/pf_ab_$v.json 2>&1
  VT_PREFILL_PAIR=1 VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf2nreg.so timeout 300 python tools/kernel_bench.py --which prefill --iters 64 >> $O/pf_ab_nreg.json 2>&1
done
VT_PREFILL_PAIR=1 VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf2trace.so timeout 300 python tools/trace_pair.py > $O/trace_pair.txt 2>&1; echo "trace rc=$?" >> $O/status
VT_PREFILL_PAIR=1 VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf2nregtrace.so timeout 300 python tools/trace_pair.py > $O/trace_pair_nreg.txt 2>&1; echo "trace nreg rc=$?" >> $O/status
cat $O/status
# sustained growth (config 2, 1000 steps past the warm free list): how the
# host waits for its oldest queued step, and chained vs plain decode layers
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline --steps 1000"
for rep in 1 2; do
  for hs in spin poll block; do
    timeout 600 $B --host-sync $hs > $O/hs_${hs}_$rep.json 2> $O/hs_${hs}_$rep.err; echo "hs $hs $rep rc=$?" >> $O/status
  done
  timeout 600 $B --host-sync poll --no-chain > $O/hs_poll_nochain_$rep.json 2> $O/hs_poll_nochain_$rep.err; echo "poll nochain $rep rc=$?" >> $O/status
done
cat $O/status
