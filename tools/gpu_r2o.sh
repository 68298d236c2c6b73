#!/bin/bash
# round 2: bounded host run-ahead (--max-ahead, default 2) vs unbounded under
# sustained growth; twins with every chunk pre-mapped.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2o
O=gpurun_out/r2o
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
for rep in 1 2; do
  timeout 600 $B --steps 2000 > $O/ma2_$rep.json 2> $O/ma2_$rep.err; echo "ma2 $rep rc=$?" >> $O/status
  VT_SETACCESS_RUNS=1 timeout 600 $B --steps 2000 > $O/ma2_runs_$rep.json 2> $O/ma2_runs_$rep.err; echo "ma2 runs $rep rc=$?" >> $O/status
done
timeout 600 $B --steps 2000 --max-ahead 0 > $O/ma0.json 2> $O/ma0.err; echo "ma0 rc=$?" >> $O/status
timeout 600 $B --steps 2000 --premap > $O/ma2_premap.json 2> $O/ma2_premap.err; echo "ma2 premap rc=$?" >> $O/status
timeout 900 $B --growth > $O/growth_ma2.json 2> $O/growth_ma2.err; echo "growth ma2 rc=$?" >> $O/status
timeout 900 $B --growth --premap > $O/growth_ma2_premap.json 2> $O/growth_ma2_premap.err; echo "growth ma2 premap rc=$?" >> $O/status
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/status
cat $O/status
