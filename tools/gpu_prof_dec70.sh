# ncu --set full of the tcgen05 decode kernel at the 70B shape (G=8, one 16-layer group).
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/prof_decode_tc70 python tools/kernel_bench.py --which decode --paths tcgen05 --shape 70b --splits ${SPLIT:-2048} --iters 1 --warmup 2 > gpurun_out/ncu_decode_tc70.log 2>&1; echo ncu rc=$?
timeout 300 python tools/kernel_bench.py --which decode --paths tcgen05 --shape 70b --splits 512,1024,2048,4096 --loop 2>&1 | grep kernel
