# Prefill kernel iteration: parity tests, then the config-3 kernel timing.
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q -m gpu > gpurun_out/pytest_prefill.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_prefill.log
timeout 300 python tools/kernel_bench.py --which prefill --iters 50 > gpurun_out/kbench_pf.log 2>&1; echo kbench rc=$?
grep kernel gpurun_out/kbench_pf.log || tail -5 gpurun_out/kbench_pf.log
