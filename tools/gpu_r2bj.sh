# r2bj: bare 50 MB stream in the QKV kernel's launch order (PDL=3: first ring
# at entry, the rest after griddepcontrol.wait) vs chunk size / stages.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bj; mkdir -p $O
P=tools/stream_probe
{
for pdl in 3 1; do for cfg in "144 352 16 8" "144 352 16 12" "144 352 32 4" "144 352 32 6" "144 352 64 3" "144 352 96 2" "148 342 16 8"; do timeout 60 $P $cfg $pdl; done; done
} > $O/out.txt 2>&1
cat $O/out.txt
