# r2bf: fused QKV ring-depth sensitivity (weight bytes in flight per SM):
# 6 / 7 / 8 stages of (16 KiB W + 8 KiB x), split 3, B=64.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bf; mkdir -p $O
cp paper_2407_15309_b200/libvtattn.so /tmp/normal.so
for r in 1 2; do for v in ring144 ring168 normal; do
  if [ $v = normal ]; then cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so; else cp build_variants/libvtattn_$v.so paper_2407_15309_b200/libvtattn.so; fi
  echo "== $v $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3,2 2>&1 | grep fused
done; done > $O/out.txt 2>&1
cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so
cat $O/out.txt
