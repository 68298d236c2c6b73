# Build libvtattn.so with -DVT_QKV_TRACE, print the fused-QKV per-CTA timeline
# (B=64, split 2 and split 3), then restore the normal build and time it.
cd $GRAFT_REPO_ROOT
C=paper_2407_15309_b200/csrc
SRCS=$(ls $C/*.cu)
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared"
$NVCC -DVT_QKV_TRACE -o paper_2407_15309_b200/libvtattn.so $SRCS
for args in "64 2" "64 3"; do python tools/trace_qkv.py $args | grep -v "w_issue"; done
$NVCC -o paper_2407_15309_b200/libvtattn.so $SRCS
timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 2,3 2>&1 | grep fused
