#!/bin/bash
# round 2 (re-entry): GPU tests, default bench, config-5 growth run, 2000-step config-2 vs premap
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 600 python bench.py > gpurun_out/r2b_bench_default.json 2> gpurun_out/r2b_bench_default.err
timeout 900 python bench.py --growth --no-e2e --no-prefill --no-qkv --no-cpu-baseline > gpurun_out/r2b_growth.json 2> gpurun_out/r2b_growth.err
timeout 900 python bench.py --growth --premap --no-e2e --no-prefill --no-qkv --no-cpu-baseline > gpurun_out/r2b_growth_premap.json 2> gpurun_out/r2b_growth_premap.err
timeout 900 python bench.py --steps 2000 --no-e2e --no-prefill --no-qkv --no-cpu-baseline > gpurun_out/r2b_cfg2_2000.json 2> gpurun_out/r2b_cfg2_2000.err
timeout 900 python bench.py --steps 2000 --no-e2e --no-prefill --no-qkv --no-cpu-baseline --premap > gpurun_out/r2b_cfg2_2000_premap.json 2> gpurun_out/r2b_cfg2_2000_premap.err
tail -3 gpurun_out/r2b_pytest.log
