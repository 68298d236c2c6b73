# r2bh: bulk-copy streaming rate vs CTAs / chunk / stages (tools/stream_probe.cu).
# 144 x 352 KiB ~ the QKV weight (50 MB) on 144 SMs.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bh; mkdir -p $O
P=tools/stream_probe
{
for cfg in "144 352 16 8" "144 352 16 4" "144 352 16 12" "144 352 32 6" "144 352 64 3" "148 342 16 8" "96 528 16 8" "144 352 8 16" "296 176 16 6"; do timeout 60 $P $cfg; done
} > $O/out.txt 2>&1
cat $O/out.txt
