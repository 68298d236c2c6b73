#!/bin/bash
# round 2: GPU test suite (one pytest per file, each under its own timeout so a
# hang is localised), VMM scaling probe, default bench with --check, prefill /
# QKV A/B against the previous kernels (build/*_v1.so), paged-library comparison.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ./tools/vmm_probe4 1 > $O/vmm_probe4_slab1.jsonl 2>&1; echo "probe1 rc=$?" >> $O/status
timeout 600 ./tools/vmm_probe4 32 > $O/vmm_probe4_slab32.jsonl 2>&1; echo "probe32 rc=$?" >> $O/status
for f in tests/test_*gpu*.py tests/test_bench_contract.py; do
  n=$(basename $f .py)
  timeout 1200 python -m pytest $f -m gpu -q -p no:cacheprovider -x > $O/pytest_$n.log 2>&1
  echo "$n rc=$? $(tail -1 $O/pytest_$n.log)" >> $O/status
done
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
timeout 600 python bench.py --check > $O/bench_check.json 2> $O/bench_check.err; echo "bench rc=$?" >> $O/status
for v in cur v1; do
  if [ $v = v1 ]; then export VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf_v1.so; fi
  timeout 300 python tools/kernel_bench.py --which prefill --iters 64 > $O/pf_$v.json 2>&1
  unset VT_LIB_LIBVTATTN
done
for v in cur v1; do
  if [ $v = v1 ]; then export VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkv_v1.so; fi
  timeout 300 python tools/kernel_bench.py --which qkv > $O/qkv_$v.json 2>&1
  unset VT_LIB_LIBVTATTN
done
timeout 900 python tools/paged_vs_vtensor.py > $O/paged.json 2> $O/paged.err; echo "paged rc=$?" >> $O/status
cat $O/status
