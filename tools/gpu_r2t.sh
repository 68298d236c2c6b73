#!/bin/bash
# round 2: SetAccess latency time series around bulk allocation / release (probe 7)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2t
O=gpurun_out/r2t
timeout 300 ./tools/vmm_probe7 > $O/probe7_a.jsonl 2> $O/probe7_a.err; echo "probe7 a rc=$?" >> $O/status
timeout 300 ./tools/vmm_probe7 > $O/probe7_b.jsonl 2> $O/probe7_b.err; echo "probe7 b rc=$?" >> $O/status
cat $O/status
