cd $GRAFT_REPO_ROOT
timeout 300 python tools/kernel_bench.py --splits 256,512,1024,2048 > gpurun_out/kbench.log 2>&1; echo kbench rc=$?
cat gpurun_out/kbench.log | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 2 -c 1 -o gpurun_out/prof_decode python tools/kernel_bench.py --which decode --iters 1 --warmup 2 > gpurun_out/ncu_decode.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/prof_prefill python tools/kernel_bench.py --which prefill --iters 1 --warmup 2 > gpurun_out/ncu_prefill.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_decode.log gpurun_out/ncu_prefill.log
