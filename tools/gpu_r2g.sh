#!/bin/bash
# round 2: extends under sustained growth with one driver thread (the default
# now): config-5 growth trace and a 2000-step config-2 run, each beside its
# --premap twin; the default bench; engine-trace evidence.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2g
O=gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-prefill --no-qkv --no-cpu-baseline"
timeout 900 $B --growth > $O/growth.json 2> $O/growth.err; echo "growth rc=$?" >> $O/status
timeout 900 $B --growth --premap > $O/growth_premap.json 2> $O/growth_premap.err; echo "growth_premap rc=$?" >> $O/status
timeout 900 $B --steps 2000 > $O/cfg2_2000.json 2> $O/cfg2_2000.err; echo "cfg2_2000 rc=$?" >> $O/status
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/status
timeout 900 python tests/engine_gpu_run.py gpu toy_cfg1 > $O/engine_toy_cfg1.json 2> $O/engine_toy.err; echo "engine toy rc=$?" >> $O/status
timeout 900 python tests/engine_gpu_run.py gpu reduced_preempt --check-every 64 > $O/engine_reduced_preempt.json 2> $O/engine_rp.err; echo "engine rp rc=$?" >> $O/status
cat $O/status
