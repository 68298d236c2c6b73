# All bench configurations of BASELINE.json on one B200 (+ the reference arm).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench/cfg2_default.json; echo cfg2 rc=$?
timeout 900 python bench.py --config llama3-8b-32k --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench/cfg5_32k_concurrent_extend.json; echo cfg5 rc=$?
timeout 900 python bench.py --config llama3-8b-32k --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --premap 2>&1 | tail -1 > gpurun_out/bench/cfg5_32k_premapped.json; echo cfg5p rc=$?
timeout 900 python bench.py --config llama2-70b-decode --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench/cfg4_70b_1gpu.json; echo cfg4 rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench/reference_arm.json; echo ref rc=$?
for f in gpurun_out/bench/*.json; do echo $f; cut -c1-160 $f; done
