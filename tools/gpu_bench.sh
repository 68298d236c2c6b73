cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 python -m pytest tests/test_decode_gpu.py -q -x -m gpu > gpurun_out/pytest_decode.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_decode.log; tail -2 gpurun_out/bench.log
