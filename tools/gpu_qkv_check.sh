cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_qkv_gpu.py -x -q > gpurun_out/qkv_tests.log 2>&1; echo qkv tests rc=$?
tail -3 gpurun_out/qkv_tests.log
timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16,256 --qkv-split 0,1 2>&1 | tail -9
bash tools/gpu_trace_qkv.sh 2>&1
