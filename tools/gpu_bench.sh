cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 900 python bench.py --config llama3-8b-32k --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench32k.log 2>&1; echo bench32k rc=$?
timeout 900 python bench.py --config llama3-8b-32k --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --premap > gpurun_out/bench32k_premap.log 2>&1; echo bench32kp rc=$?
tail -1 gpurun_out/pytest_gpu.log
