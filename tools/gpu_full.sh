# Round validation: GPU tests, smoke, default bench, config lines, reference arm.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 400 python bench.py --config llama2-70b-decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench70b.log 2>&1; echo b70 rc=$?
timeout 600 python bench.py --config llama3-8b-32k --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench32k.log 2>&1; echo b32k rc=$?
timeout 300 python bench.py --config toy-cfg1 --steps 20 --warmup 5 > gpurun_out/benchtoy.log 2>&1; echo btoy rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/benchref.log 2>&1; echo ref rc=$?
