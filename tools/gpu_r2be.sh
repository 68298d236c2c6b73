#!/bin/bash
# round 2 (late, after the decode p_full fix): ncu evidence per bench config. One `--set full` capture of the
# decode kernel INSIDE bench.py for each config the bench reports
# (roofline.traffic per config, tools/make_traffic.py), the cuda-core path,
# the prefill and fused-QKV kernels, and a launch list of the default step
# restricted to this package's kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2be
O=gpurun_out/r2be
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for spec in llama3-8b-decode/tcgen05 llama2-70b-decode/tcgen05 llama3-8b-32k/tcgen05 toy-cfg1/tcgen05 llama3-8b-decode/cuda_core; do
  cfg=${spec%/*}; path=${spec#*/}
  k=regex:decode_tc; [ $path = cuda_core ] && k=regex:decode_splitkv
  skip=40; [ $cfg = toy-cfg1 ] && skip=1
  timeout 900 ncu --set full --clock-control none --import-source on -k $k -s $skip -c 1 \
    -o $O/decode_${cfg}__${path} python bench.py --config $cfg --path $path --profile-steps 3 --no-cpu-baseline > $O/decode_${cfg}__${path}.log 2>&1
  echo "ncu $spec rc=$?" >> $O/status
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 3 -c 1 \
  -o $O/prefill python tools/kernel_bench.py --which prefill --iters 1 --warmup 3 > $O/prefill.log 2>&1; echo "ncu prefill rc=$?" >> $O/status
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qkv_append -s 6 -c 1 \
  -o $O/qkv python tools/kernel_bench.py --which qkv > $O/qkv.log 2>&1; echo "ncu qkv rc=$?" >> $O/status
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kv_append|decode|prefill|qkv|combine" -c 300 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1; echo "launches rc=$?" >> $O/status
cat $O/status
