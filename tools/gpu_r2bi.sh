# r2bi: bare 50 MB bulk-copy stream with programmatic dependent launch
# (PDL=1 waits on the previous launch like a layer stack; PDL=2 does not).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bi; mkdir -p $O
P=tools/stream_probe
{
for pdl in 0 1 2; do for cfg in "144 352 16 8" "148 342 16 8" "144 352 64 3"; do timeout 60 $P $cfg $pdl; done; done
} > $O/out.txt 2>&1
cat $O/out.txt
