# Final round-2 validation of HEAD: GPU suite, smoke, default bench, reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final_r2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 400 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python bench.py --impl reference > $O/benchref.log 2>&1; echo ref rc=$?
