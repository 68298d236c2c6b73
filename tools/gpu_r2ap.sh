#!/bin/bash
# round 2 (late): does mapping in flight slow the decode launches? default vs
# --premap (same box, alternated), kernel_bench chained; then the config-5
# growth trace and 2000-step sustained config 2, each with its pre-mapped twin
cd "$(dirname "$0")/.."
O=gpurun_out/r2ap; mkdir -p $O
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
for r in 1 2; do
  timeout 600 $B > $O/default_$r.json 2>> $O/err; echo "default $r rc=$?" >> $O/status
  timeout 600 $B --premap > $O/premap_$r.json 2>> $O/err; echo "premap $r rc=$?" >> $O/status
done
timeout 300 python tools/kernel_bench.py --which decode --paths tcgen05 --splits 2048 --loop --chained --iters 40 > $O/kb.txt 2>> $O/err
timeout 1500 $B --growth > $O/growth.json 2>> $O/err; echo "growth rc=$?" >> $O/status
timeout 1500 $B --growth --premap > $O/growth_premap.json 2>> $O/err; echo "growth premap rc=$?" >> $O/status
timeout 900 $B --steps 2000 > $O/sustained.json 2>> $O/err; echo "sustained rc=$?" >> $O/status
timeout 900 $B --steps 2000 --premap > $O/sustained_premap.json 2>> $O/err; echo "sustained premap rc=$?" >> $O/status
cat $O/status $O/kb.txt
for f in $O/*.json; do tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d.get('extend',{}); r=d['roofline']
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], d['steps'], r['per_launch_us'], {k:e.get(k) for k in ['hidden','host_waited_steps','gpu_stalled_steps','chunks_mapped']})"; done
