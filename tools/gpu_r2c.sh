#!/bin/bash
# round 2: full GPU test suite, default bench with --check, prefill/QKV A/B
# against the previous kernels (build/*_v1.so), paged-library comparison, ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log
timeout 600 python bench.py --check > gpurun_out/r2c_bench_check.json 2> gpurun_out/r2c_bench_check.err
for v in cur v1; do
  if [ $v = v1 ]; then export VT_LIB_LIBVTATTN=$PWD/build/libvtattn_pf_v1.so; fi
  timeout 300 python tools/kernel_bench.py --which prefill --iters 64 > gpurun_out/r2c_pf_$v.json 2>&1
  unset VT_LIB_LIBVTATTN
done
for v in cur v1; do
  if [ $v = v1 ]; then export VT_LIB_LIBVTATTN=$PWD/build/libvtattn_qkv_v1.so; fi
  timeout 300 python tools/kernel_bench.py --which qkv > gpurun_out/r2c_qkv_$v.json 2>&1
  unset VT_LIB_LIBVTATTN
done
timeout 900 python tools/paged_vs_vtensor.py > gpurun_out/r2c_paged.json 2> gpurun_out/r2c_paged.err
tail -3 gpurun_out/r2c_pytest.log
