# r2at: fused QKV, separate L2 prefetch depths for the pair CTAs (enter as the
# previous launch's pairs leave: HBM idle) and the helpers (enter while the
# previous pairs still stream), swept with the helper share.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2at; mkdir -p $O
run() { echo "== pair $1 helper $2 q64 $3"; VT_QKV_L2_PREFETCH=$1 VT_QKV_L2_PREFETCH_HELPER=$2 VT_QKV_HELPER_Q64=$3 timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3 2>&1 | grep fused; }
{
run 4 4 16
run 8 0 16
run 8 4 16
run 16 0 16
run 16 4 16
run 16 0 12
run 16 0 14
run 16 4 14
run 12 2 14
run 8 2 14
run 4 4 16
} > $O/sweep.txt 2>&1
grep -A1 '^==' $O/sweep.txt | grep -v '^--' | paste - - | sed 's/{"kernel.*"us": \([0-9.]*\),.*frac_of_hbm": \([0-9.]*\)}/\1 \2/'
