#!/bin/bash
# round 2: GPU tests + default bench + a 2000-step growth-bound config-2 run
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py > gpurun_out/r2a_bench_default.json 2> gpurun_out/r2a_bench_default.err
timeout 900 python bench.py --steps 2000 --no-e2e --no-prefill --no-qkv --no-cpu-baseline > gpurun_out/r2a_cfg2_2000.json 2> gpurun_out/r2a_cfg2_2000.err
timeout 900 python bench.py --steps 2000 --no-e2e --no-prefill --no-qkv --no-cpu-baseline --phys-reserve 0 > gpurun_out/r2a_cfg2_2000_noreserve.json 2>&1
timeout 900 python bench.py --steps 2000 --no-e2e --no-prefill --no-qkv --no-cpu-baseline --premap > gpurun_out/r2a_cfg2_2000_premap.json 2>&1
tail -3 gpurun_out/r2a_pytest.log
