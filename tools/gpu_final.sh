# Round-end validation: GPU tests, smoke, default bench, reference arm, a 2-rank torchrun run.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/benchref.log 2>&1; echo ref rc=$?
VT_BENCH_HANG_DUMP_S=250 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_tr2.log 2>&1; echo tr2 rc=$?
tail -1 gpurun_out/bench_tr2.log | cut -c1-300
