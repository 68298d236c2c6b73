# r2bd: does the fused QKV's scattered K/V row-store tail (64 requests' VA
# pages) set the launch-to-launch latency? Timing-only builds without the K/V
# row stores / without any row stores vs the product build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bd; mkdir -p $O
cp paper_2407_15309_b200/libvtattn.so /tmp/normal.so
for r in 1 2; do for v in normal nokv nostore; do
  if [ $v = normal ]; then cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so; else cp build_variants/libvtattn_$v.so paper_2407_15309_b200/libvtattn.so; fi
  echo "== $v $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3 2>&1 | grep fused
done; done > $O/out.txt 2>&1
cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so
cat $O/out.txt
