#!/bin/bash
# round 2: ncu evidence. Launch list of the default bench step, and one
# `--set full` capture of the decode kernel INSIDE bench.py for each config the
# bench reports (roofline.traffic per config), plus prefill and fused QKV.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1; echo "launches rc=$?"
for cfg in llama3-8b-decode llama2-70b-decode llama3-8b-32k toy-cfg1; do
  skip=40; [ $cfg = toy-cfg1 ] && skip=1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s $skip -c 1 \
    -o $O/decode_$cfg python bench.py --config $cfg --profile-steps 3 --no-cpu-baseline > $O/decode_$cfg.log 2>&1
  echo "ncu $cfg rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 3 -c 1 \
  -o $O/prefill python tools/kernel_bench.py --which prefill --iters 1 --warmup 3 > $O/prefill.log 2>&1; echo "ncu prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qkv_append -s 6 -c 1 \
  -o $O/qkv python tools/kernel_bench.py --which qkv > $O/qkv.log 2>&1; echo "ncu qkv rc=$?"
ls -la $O
