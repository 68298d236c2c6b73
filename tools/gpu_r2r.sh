#!/bin/bash
# round 2: what sets cuMemSetAccess cost under load (probe 6), and the bench's
# sustained-growth run unchained / without the physical reserve
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2r
O=gpurun_out/r2r
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ./tools/vmm_probe6 > $O/probe6.jsonl 2> $O/probe6.err; echo "probe6 rc=$?" >> $O/status
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline --steps 1000"
for rep in 1 2; do
  timeout 600 $B --no-chain > $O/nochain_$rep.json 2> $O/nochain_$rep.err; echo "nochain $rep rc=$?" >> $O/status
  timeout 600 $B > $O/chain_$rep.json 2> $O/chain_$rep.err; echo "chain $rep rc=$?" >> $O/status
  timeout 600 $B --phys-reserve 0 > $O/noreserve_$rep.json 2> $O/noreserve_$rep.err; echo "noreserve $rep rc=$?" >> $O/status
done
cat $O/status
