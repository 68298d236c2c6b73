cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 900 python bench.py --config llama2-70b-decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench70.log 2>&1; echo bench70 rc=$?
tail -2 gpurun_out/bench.log | cut -c1-1500; tail -3 gpurun_out/bench70.log | cut -c1-1800
