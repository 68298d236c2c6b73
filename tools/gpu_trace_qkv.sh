# Build libvtattn.so with -DVT_QKV_TRACE, print the fused-QKV per-CTA timeline
# (B=64 and B=256 by default), then restore the normal build and time it.
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
SRCS="$C/vt_decode.cu $C/vt_decode_tc.cu $C/vt_kvops.cu $C/vt_prefill.cu $C/vt_qkv.cu $C/vt_tmap.cu"
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared"
$NVCC -DVT_QKV_TRACE -o paper_2407_15309_b200/libvtattn.so $SRCS
for args in "64 0" "256 0"; do python tools/trace_qkv.py $args | grep -v "entry\|setup\|w_issue\|first_land"; done
$NVCC -o paper_2407_15309_b200/libvtattn.so $SRCS
timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 0 2>&1 | grep fused
