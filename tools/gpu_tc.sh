cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -m gpu > gpurun_out/pytest_decode.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_decode.log
timeout 300 python tools/kernel_bench.py --which decode --splits 2048 --loop > gpurun_out/kbench.log 2>&1; echo kbench rc=$?
timeout 300 python tools/kernel_bench.py --which decode --splits 2048 --loop --shape 70b >> gpurun_out/kbench.log 2>&1; echo kbench rc=$?
cat gpurun_out/kbench.log | grep kernel
