#!/bin/bash
# round 2: full GPU suite at HEAD; growth trace with the time-based lead (x2) and its
# pre-mapped twin; sustained config 2 (2000 steps); default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2ab
O=gpurun_out/r2ab
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?" >> $O/status
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
for rep in 1 2; do
  timeout -s INT 1200 $B --growth > $O/growth_$rep.json 2> $O/growth_$rep.err; echo "growth $rep rc=$?" >> $O/status
done
timeout -s INT 1800 $B --growth --premap > $O/growth_premap.json 2> $O/growth_premap.err; echo "growth premap rc=$?" >> $O/status
timeout -s INT 900 $B --steps 2000 > $O/sustained.json 2> $O/sustained.err; echo "sustained rc=$?" >> $O/status
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/status
cat $O/status
