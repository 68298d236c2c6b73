# r2bg: decode split sweep inside the default bench step (lens 4033..4121 over
# the run: 32-33 tiles per request) vs the auto choice (2176 here).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bg; mkdir -p $O
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
for r in 1 2; do for s in 0 2048 1536 1408 1152 2304; do
  timeout 300 $B --split $s > $O/s${s}_$r.json 2>> $O/err
  tail -1 $O/s${s}_$r.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split $s rep $r', d['value'], d['ms_per_step'], d['roofline']['per_launch_us'])"
done; done > $O/out.txt 2>&1
cat $O/out.txt
