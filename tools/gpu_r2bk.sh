# r2bk: fused QKV with paired 32 KiB weight copies (weight blocks side by side
# in the ring) vs the 16 KiB-copy build: QKV tests, then A/B kernel bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bk; mkdir -p $O
cp paper_2407_15309_b200/libvtattn.so /tmp/new.so
{
timeout 600 python -m pytest tests/test_qkv_gpu.py -q -x 2>&1 | tail -2
for r in 1 2 3; do for v in new single16k; do
  if [ $v = new ]; then cp /tmp/new.so paper_2407_15309_b200/libvtattn.so; else cp build_variants/libvtattn_$v.so paper_2407_15309_b200/libvtattn.so; fi
  echo "== $v $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16 --qkv-split 3,2 2>&1 | grep fused
done; done
} > $O/out.txt 2>&1
cp /tmp/new.so paper_2407_15309_b200/libvtattn.so
cat $O/out.txt
