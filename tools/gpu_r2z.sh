#!/bin/bash
# round 2: config 4 (70B, one GPU) over 400 steps: extends in flight (lead 3 / 24) vs pre-mapped
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2z
O=gpurun_out/r2z
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline --config llama2-70b-decode --steps 400"
timeout 900 $B --lead-chunks 3 > $O/cfg4_400_lead3.json 2> $O/cfg4_400_lead3.err; echo "lead3 rc=$?" >> $O/status
timeout 900 $B > $O/cfg4_400_lead24.json 2> $O/cfg4_400_lead24.err; echo "lead24 rc=$?" >> $O/status
timeout 900 $B --premap > $O/cfg4_400_premap.json 2> $O/cfg4_400_premap.err; echo "premap rc=$?" >> $O/status
timeout 900 $B --no-chain > $O/cfg4_400_lead24_nochain.json 2> $O/cfg4_400_lead24_nochain.err; echo "nochain rc=$?" >> $O/status
cat $O/status
