#!/bin/bash
# round 2: config 4 step time vs lead / run-ahead; sustained growth vs driver threads
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2y
O=gpurun_out/r2y
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
timeout 600 $B --config llama2-70b-decode --lead-chunks 3 > $O/cfg4_lead3.json 2> $O/cfg4_lead3.err; echo "cfg4 lead3 rc=$?" >> $O/status
timeout 600 $B --config llama2-70b-decode > $O/cfg4_lead24.json 2> $O/cfg4_lead24.err; echo "cfg4 lead24 rc=$?" >> $O/status
timeout 600 $B --config llama2-70b-decode --max-ahead 0 > $O/cfg4_lead24_ma0.json 2> $O/cfg4_lead24_ma0.err; echo "cfg4 lead24 ma0 rc=$?" >> $O/status
timeout 600 $B --config llama2-70b-decode --lead-chunks 3 --max-ahead 0 > $O/cfg4_lead3_ma0.json 2> $O/cfg4_lead3_ma0.err; echo "cfg4 lead3 ma0 rc=$?" >> $O/status
for rep in 1 2; do
  for t in 1 2 4; do
    timeout 600 $B --steps 1000 --driver-threads $t > $O/sus_thr${t}_$rep.json 2> $O/sus_thr${t}_$rep.err; echo "sus thr$t $rep rc=$?" >> $O/status
  done
done
cat $O/status
