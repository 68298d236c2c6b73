# Build libvtattn.so with -DVT_PF_TRACE and print the prefill timeline of one CTA.
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared -DVT_PF_TRACE $EXTRA -o paper_2407_15309_b200/libvtattn.so $C/vt_decode.cu $C/vt_decode_tc.cu $C/vt_kvops.cu $C/vt_prefill.cu $C/vt_qkv.cu $C/vt_tmap.cu
python tools/trace_prefill.py
