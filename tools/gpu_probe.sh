cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_vmm.py > gpurun_out/probe_vmm.json 2> gpurun_out/probe_vmm.err; echo probe rc=$?
cat gpurun_out/probe_vmm.json; tail -5 gpurun_out/probe_vmm.err
