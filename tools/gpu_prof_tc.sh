cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/prof_decode_tc python tools/kernel_bench.py --which decode --paths tcgen05 --splits 2048 --iters 1 --warmup 2 > gpurun_out/ncu_decode_tc.log 2>&1; echo ncu rc=$?
