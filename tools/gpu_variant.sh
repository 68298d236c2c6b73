# Build libvtattn.so with each given nvcc flag set and time the config-3 prefill.
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
for V in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared $V -o paper_2407_15309_b200/libvtattn.so $C/vt_decode.cu $C/vt_decode_tc.cu $C/vt_kvops.cu $C/vt_prefill.cu $C/vt_tmap.cu
  echo "=== variant $V"; python tools/debug_prefill.py 2>&1 | grep -E "case" | head -1
  timeout 300 python tools/kernel_bench.py --which prefill --iters 30 2>&1 | grep -oE '"TFLOP/s": [0-9.]+'
done
