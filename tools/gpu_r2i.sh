#!/bin/bash
# round 2 (session 3): P-in-shared-memory prefill (parity + A/B vs the previous
# kernel), extra plain kernel boundaries for the driver's VMM work under
# sustained growth, and the engine-on-GPU traces (reference engine now present).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2i
O=gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_poisoned_tails_gpu.py -x -q > $O/pytest_prefill.log 2>&1; echo "pytest prefill rc=$?" >> $O/status
for v in cur old cur old; do
  if [ $v = old ]; then export VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pfold.so; fi
  timeout 300 python tools/kernel_bench.py --which prefill --iters 64 >> $O/pf_ab_$v.json 2>&1
  unset VT_LIB_LIBVTATTN
done
echo "pf ab done" >> $O/status
timeout 300 python tools/kernel_bench.py --which prefill --iters 32 --pf-prefix 8192 > $O/pf_8k.json 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
for pe in 0 8 4; do
  timeout 600 $B --steps 2000 --plain-every $pe > $O/cfg2_2000_pe$pe.json 2> $O/cfg2_2000_pe$pe.err; echo "cfg2_2000 pe=$pe rc=$?" >> $O/status
done
timeout 600 $B --steps 2000 --plain-every 4 --plain-adaptive > $O/cfg2_2000_pe4a.json 2> $O/cfg2_2000_pe4a.err; echo "cfg2_2000 pe4a rc=$?" >> $O/status
timeout 600 $B --steps 2000 --plain-every 8 --premap > $O/cfg2_2000_pe8_premap.json 2> $O/cfg2_2000_pe8_premap.err; echo "cfg2_2000 pe8 premap rc=$?" >> $O/status
timeout 600 $B --steps 2000 --premap > $O/cfg2_2000_premap.json 2> $O/cfg2_2000_premap.err; echo "cfg2_2000 premap rc=$?" >> $O/status
timeout 900 $B --growth --plain-every 8 > $O/growth_pe8.json 2> $O/growth_pe8.err; echo "growth pe8 rc=$?" >> $O/status
timeout 1800 python -m pytest tests/test_engine_gpu.py -x -q > $O/pytest_engine.log 2>&1; echo "pytest engine rc=$?" >> $O/status
cat $O/status
