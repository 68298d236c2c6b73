cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -m gpu -k paged > gpurun_out/pytest_paged.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_paged.log
timeout 600 python tools/paged_vs_vtensor.py > gpurun_out/paged.json 2> gpurun_out/paged.err; echo paged rc=$?
cat gpurun_out/paged.json; tail -3 gpurun_out/paged.err
