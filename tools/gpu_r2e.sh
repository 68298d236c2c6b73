#!/bin/bash
# round 2: what makes cuMemSetAccess 10x slower inside the bench than in the
# standalone probe? 300-step config-2 runs varying one factor at a time, the
# context probe, and the engine traces.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2e
O=gpurun_out/r2e
timeout 300 ./tools/vmm_probe5 > $O/vmm_probe5.jsonl 2>&1; echo "probe5 rc=$?" >> $O/status
B="python bench.py --steps 300 --warmup 5 --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
timeout 400 $B > $O/cfg2_300_default.json 2> $O/cfg2_300_default.err; echo "default rc=$?" >> $O/status
timeout 400 $B --no-chain > $O/cfg2_300_nochain.json 2> $O/cfg2_300_nochain.err; echo "nochain rc=$?" >> $O/status
timeout 400 $B --driver-threads 1 > $O/cfg2_300_thr1.json 2> $O/cfg2_300_thr1.err; echo "thr1 rc=$?" >> $O/status
timeout 400 $B --no-chain --driver-threads 1 > $O/cfg2_300_nochain_thr1.json 2> $O/cfg2_300_nochain_thr1.err; echo "nochain_thr1 rc=$?" >> $O/status
timeout 400 $B --path cuda_core > $O/cfg2_300_cudacore.json 2> $O/cfg2_300_cudacore.err; echo "cudacore rc=$?" >> $O/status
timeout 400 $B --phys-reserve 0 > $O/cfg2_300_noreserve.json 2> $O/cfg2_300_noreserve.err; echo "noreserve rc=$?" >> $O/status
timeout 2400 python -m pytest tests/test_engine_gpu.py -m gpu -q -p no:cacheprovider > $O/pytest_engine.log 2>&1; echo "engine rc=$? $(tail -1 $O/pytest_engine.log)" >> $O/status
cat $O/status
