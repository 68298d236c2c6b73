cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multirank_gpu.py -x -q > gpurun_out/mr_gpu.log 2>&1; echo mr rc=$?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --config llama2-70b-decode > gpurun_out/bench_tr2.log 2>&1; echo tr2 rc=$?
tail -3 gpurun_out/mr_gpu.log
