cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest $VT_TESTS -x -q -m gpu > gpurun_out/pytest_one.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_one.log
