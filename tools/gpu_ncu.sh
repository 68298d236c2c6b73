cd $GRAFT_REPO_ROOT
# launch list of the bench command (cold, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/prof_decode_tc python tools/kernel_bench.py --which decode --paths tcgen05 --splits 2048 --iters 1 --warmup 2 > gpurun_out/ncu_decode_tc.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 2 -c 1 -o gpurun_out/prof_decode_cc python tools/kernel_bench.py --which decode --paths cuda_core --splits 1024 --iters 1 --warmup 2 > gpurun_out/ncu_decode_cc.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/prof_prefill python tools/kernel_bench.py --which prefill --iters 1 --warmup 2 > gpurun_out/ncu_prefill.log 2>&1; echo ncu3 rc=$?
