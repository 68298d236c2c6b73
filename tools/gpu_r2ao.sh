#!/bin/bash
# round 2: decode split-size sweep, 32 chained layers (config 2 shape)
cd "$(dirname "$0")/.."
O=gpurun_out/r2ao; mkdir -p $O
for r in 1 2; do
timeout 300 python tools/kernel_bench.py --which decode --paths tcgen05 --splits 1024,1408,2048,4096 --loop --chained --iters 40 2>>$O/err | tee -a $O/sweep.txt
done
