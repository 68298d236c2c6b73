# Build libvtattn.so with each given nvcc flag set and run $VARIANT_CMD (default: config-3 prefill timing).
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
for V in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared $V -o paper_2407_15309_b200/libvtattn.so $C/*.cu
  echo "=== variant $V"
  eval "${VARIANT_CMD:-timeout 300 python tools/kernel_bench.py --which prefill --iters 30}" 2>&1 | grep -E "kernel|Error"
done
