# Full GPU check: tests, default bench line, qkv ncu capture.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
QKV_SPLIT=0 bash tools/gpu_prof_qkv.sh
