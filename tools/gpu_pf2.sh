cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_prefill_gpu.py tests/test_prefix_share_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/kernel_bench.py --which prefill 2>&1 | tail -3
bash tools/gpu_trace_pf.sh 2>&1 | tail -5
