#!/bin/bash
# round 2: extends 24 chunks ahead by default — default bench line, sustained
# growth (config 2, 2000 steps) and the config-5 growth trace, each with its
# pre-mapped twin; config 4 on one GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2x
O=gpurun_out/r2x
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/status
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
timeout 900 $B --steps 2000 > $O/sustained.json 2> $O/sustained.err; echo "sustained rc=$?" >> $O/status
timeout 900 $B --steps 2000 --premap > $O/sustained_premap.json 2> $O/sustained_premap.err; echo "sustained premap rc=$?" >> $O/status
timeout 1200 $B --growth > $O/growth.json 2> $O/growth.err; echo "growth rc=$?" >> $O/status
timeout 1200 $B --growth --premap > $O/growth_premap.json 2> $O/growth_premap.err; echo "growth premap rc=$?" >> $O/status
timeout 900 $B --config llama2-70b-decode > $O/cfg4.json 2> $O/cfg4.err; echo "cfg4 rc=$?" >> $O/status
timeout 900 $B --config llama3-8b-32k > $O/cfg5.json 2> $O/cfg5.err; echo "cfg5 rc=$?" >> $O/status
cat $O/status
