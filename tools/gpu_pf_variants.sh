# A/B prefill variants (compile flags) on config 3: kernel_bench TFLOP/s + trace period.
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
for flags in ${VARIANTS:-"-DVT_PF_X"}; do
  echo "== $flags"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared ${flags//,/ } -o paper_2407_15309_b200/libvtattn.so $C/vt_decode.cu $C/vt_decode_tc.cu $C/vt_kvops.cu $C/vt_prefill.cu $C/vt_qkv.cu $C/vt_tmap.cu
  timeout 120 python tools/kernel_bench.py --which prefill 2>&1 | tail -1
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared -DVT_PF_TRACE ${flags//,/ } -o paper_2407_15309_b200/libvtattn.so $C/vt_decode.cu $C/vt_decode_tc.cu $C/vt_kvops.cu $C/vt_prefill.cu $C/vt_qkv.cu $C/vt_tmap.cu
  timeout 120 python tools/trace_prefill.py 2>&1 | tail -3
done
