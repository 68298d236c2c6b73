cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -m gpu > gpurun_out/pytest_decode.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_decode.log
timeout 300 python tools/kernel_bench.py --which decode --splits 512,1024,2048 > gpurun_out/kbench.log 2>&1; echo kbench rc=$?
timeout 300 python tools/kernel_bench.py --which decode --splits 1024,2048,4096 --loop >> gpurun_out/kbench.log 2>&1; echo kbench rc=$?
cat gpurun_out/kbench.log | tail -14
