#!/bin/bash
# round 2 (session 3): GPU test suite, then the r2g growth/sustained runs with
# one driver thread, then the bench launch list under ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2h
O=gpurun_out/r2h
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
bash tools/gpu_r2g.sh > $O/r2g.log 2>&1; echo "r2g rc=$?" >> $O/status
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-prefill --no-qkv > $O/launches_bench.log 2>&1; echo "launches rc=$?" >> $O/status
cat $O/status
