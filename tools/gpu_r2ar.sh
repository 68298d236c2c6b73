# r2ar: fused QKV start-up: release vs relaxed cluster arrive (trace in a CUDA
# graph of 9 back-to-back launches, rotating or one weight) + kernel bench A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ar; mkdir -p $O
V=build_variants
for v in rel_trace rlx_trace rel rlx; do
  cp $V/libvtattn_$v.so paper_2407_15309_b200/libvtattn.so
  case $v in
    *_trace) for args in "64 3 chain graph" "64 3 chain same" "64 2 chain graph"; do
               echo "== $v $args"; timeout 120 python tools/trace_qkv.py $args | grep -v w_issue; done ;;
    *) for r in 1 2; do echo "== $v run $r"; timeout 300 python tools/kernel_bench.py --which qkv --qkv-batch 64,16 --qkv-split 2,3 2>&1 | grep fused; done ;;
  esac
done > $O/out.txt 2>&1
cp $V/libvtattn_rlx.so paper_2407_15309_b200/libvtattn.so
timeout 900 python -m pytest tests/test_qkv_gpu.py -x -q >> $O/out.txt 2>&1
tail -3 $O/out.txt
