# r2as: fused QKV with an L2 prefetch of the weight blocks past the first ring
# (VT_QKV_L2_PREFETCH), swept with the helper share (VT_QKV_HELPER_Q64);
# kernel bench (CUDA graph of 20 launches, 4 rotating weights) + traces.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2as; mkdir -p $O
for pf in 0 4 8 16 64; do for hq in 16 20 24; do
  echo "== pf $pf helper_q64 $hq"
  VT_QKV_L2_PREFETCH=$pf VT_QKV_HELPER_Q64=$hq timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3 2>&1 | grep fused
done; done > $O/sweep.txt 2>&1
for pf in 0 4 8 64; do echo "== split2 pf $pf"; VT_QKV_L2_PREFETCH=$pf timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 2 2>&1 | grep fused; done >> $O/sweep.txt 2>&1
cp paper_2407_15309_b200/libvtattn.so /tmp/normal.so
cp build_variants/libvtattn_trace.so paper_2407_15309_b200/libvtattn.so
for pf in 0 64; do echo "== trace pf $pf"; VT_QKV_L2_PREFETCH=$pf timeout 120 python tools/trace_qkv.py 64 3 chain graph | grep -v w_issue; done > $O/trace.txt 2>&1
cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so
cat $O/sweep.txt
