#!/bin/bash
# round 2: the CTA-pair prefill kernel (vt_prefill_pair.cu, VT_PREFILL_PAIR=1):
# parity first (short timeout: a wrong barrier protocol hangs), then A/B
# against the single-CTA kernel on config 3 and the 8k-prefix shape.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2l
O=gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VT_PREFILL_PAIR=1 timeout 120 python tools/kernel_bench.py --which prefill --iters 2 --warmup 1 > $O/pair_smoke.json 2>&1; echo "pair smoke rc=$?" >> $O/status
if grep -q "rc=0" $O/status; then
  VT_PREFILL_PAIR=1 timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_poisoned_tails_gpu.py -x -q > $O/pytest_pair.log 2>&1; echo "pytest pair rc=$?" >> $O/status
  for v in 1 0 1 0; do
    VT_PREFILL_PAIR=$v timeout 300 python tools/kernel_bench.py --which prefill --iters 64 >> $O/pf_ab_$v.json 2>&1
  done
  for v in 1 0; do
    VT_PREFILL_PAIR=$v timeout 300 python tools/kernel_bench.py --which prefill --iters 16 --pf-prefix 8192 >> $O/pf_8k_$v.json 2>&1
  done
  VT_PREFILL_PAIR=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_pair -s 3 -c 1 \
    -o $O/prefill_pair python tools/kernel_bench.py --which prefill --iters 1 --warmup 3 > $O/ncu_pair.log 2>&1; echo "ncu pair rc=$?" >> $O/status
fi
cat $O/status
