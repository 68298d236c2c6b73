# r2aq: steady-state (back-to-back PDL) timeline of the fused QKV kernel with
# setup sub-points; then the normal build, kernel bench and a default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=paper_2407_15309_b200/csrc
SRCS=$(ls $C/*.cu)
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared"
cp paper_2407_15309_b200/libvtattn.so /tmp/libvtattn_normal.so
$NVCC -DVT_QKV_TRACE -o paper_2407_15309_b200/libvtattn.so $SRCS
for args in "64 3 chain" "64 3" "64 2 chain"; do timeout 120 python tools/trace_qkv.py $args | grep -v "w_issue"; done > gpurun_out/r2aq_trace.txt 2>&1
cp /tmp/libvtattn_normal.so paper_2407_15309_b200/libvtattn.so
timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3 2>&1 | grep fused >> gpurun_out/r2aq_trace.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2aq_bench.json 2> gpurun_out/r2aq_bench.err
tail -c 600 gpurun_out/r2aq_bench.err
