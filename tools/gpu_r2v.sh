#!/bin/bash
# round 2: sustained growth vs in-process NVML clock sampling rate; what else runs on the box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2v
O=gpurun_out/r2v
ps -eo pid,ppid,pcpu,etime,args > $O/ps.txt 2>&1
nvidia-smi -q -d PERFORMANCE,CLOCK > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline --steps 1000"
for rep in 1 2 3; do
  timeout 600 $B --clock-interval 1.0 > $O/ci1_$rep.json 2> $O/ci1_$rep.err; echo "ci 1.0 $rep rc=$?" >> $O/status
  timeout 600 $B --clock-interval 0.05 > $O/ci005_$rep.json 2> $O/ci005_$rep.err; echo "ci 0.05 $rep rc=$?" >> $O/status
done
ps -eo pid,ppid,pcpu,etime,args > $O/ps_end.txt 2>&1
cat $O/status
