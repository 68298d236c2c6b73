#!/bin/bash
# round 2: sustained growth vs how far ahead requests are extended; host steal time
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2w
O=gpurun_out/r2w
nproc > $O/host.txt; cat /proc/cpuinfo | grep "model name" | head -1 >> $O/host.txt; uptime >> $O/host.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline --steps 1000"
for rep in 1 2; do
  for lead in 3 12 24; do
    head -1 /proc/stat > $O/stat_${lead}_$rep.txt
    timeout 600 $B --lead-chunks $lead > $O/lead${lead}_$rep.json 2> $O/lead${lead}_$rep.err; echo "lead $lead $rep rc=$?" >> $O/status
    head -1 /proc/stat >> $O/stat_${lead}_$rep.txt
  done
done
cat $O/status
