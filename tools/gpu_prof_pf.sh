# ncu --set full of the prefill kernel (config 3), one launch, with source.
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/prof_prefill python tools/kernel_bench.py --which prefill --iters 1 --warmup 2 > gpurun_out/ncu_prefill.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_prefill.log
