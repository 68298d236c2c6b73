# r2av: is the fused QKV stream bound by SM ingest of x? Timing-only variant
# that reads x in the first ring only (wrong results) vs the product build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2av; mkdir -p $O
cp paper_2407_15309_b200/libvtattn.so /tmp/normal.so
for r in 1 2; do
  for v in normal nox; do
    if [ $v = nox ]; then cp build_variants/libvtattn_nox.so paper_2407_15309_b200/libvtattn.so; else cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so; fi
    echo "== $v $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 2,3 2>&1 | grep fused
  done
done > $O/out.txt 2>&1
cp /tmp/normal.so paper_2407_15309_b200/libvtattn.so
cat $O/out.txt
