#!/bin/bash
# round 2: split 3 by default (per-stream workspace): QKV + ABI tests, kernel bench, bench.py, smoke
cd "$(dirname "$0")/.."
O=gpurun_out/r2ak; mkdir -p $O
timeout 600 python -m pytest tests/test_qkv_gpu.py tests/test_abi_errors_gpu.py tests/test_serving_gpu.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/status
tail -2 $O/tests.log
timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16 --qkv-split 0,2,3 2>>$O/kb.err | grep fused > $O/kb.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status
cat $O/status $O/kb.txt; tail -1 $O/smoke.log
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['qkv_append']))"
