cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r2ak
timeout 900 python -m pytest tests/test_qkv_gpu.py tests/test_abi_errors_gpu.py tests/test_serving_gpu.py tests/test_engine_gpu.py tests/test_bench_check_gpu.py -q > gpurun_out/r2ak/tests2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2ak/tests2.log
