cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multirank_gpu.py tests/test_decode_gpu.py -x -q > gpurun_out/mr_gpu.log 2>&1; echo mr rc=$?
VT_BENCH_HANG_DUMP_S=150 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --config llama2-70b-decode --no-prefill --no-qkv > gpurun_out/bench_tr2.log 2>&1; echo tr2 rc=$?
tail -3 gpurun_out/mr_gpu.log
