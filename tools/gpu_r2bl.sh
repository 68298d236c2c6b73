# r2bl: fused QKV with prefetch.tensormap of x's descriptor at entry vs HEAD.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bl; mkdir -p $O
{
cp build_variants/libvtattn_xpf.so paper_2407_15309_b200/libvtattn.so
timeout 600 python -m pytest tests/test_qkv_gpu.py -q -x 2>&1 | tail -1
for r in 1 2 3; do for v in xpf base; do
  cp build_variants/libvtattn_$v.so paper_2407_15309_b200/libvtattn.so
  echo "== $v $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16 --qkv-split 3 2>&1 | grep fused
done; done
} > $O/out.txt 2>&1
cp build_variants/libvtattn_xpf.so paper_2407_15309_b200/libvtattn.so
cat $O/out.txt
