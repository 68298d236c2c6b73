# ncu --set full of the fused QKV + KV append kernel (Llama-3-8B, B=64).
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qkv_append -s 6 -c 1 -o gpurun_out/prof_qkv python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split ${QKV_SPLIT:-2} > gpurun_out/ncu_qkv.log 2>&1; echo ncu rc=$?
