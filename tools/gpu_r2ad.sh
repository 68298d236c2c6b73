#!/bin/bash
# round 2: config-2 decode, tcgen05 vTensor kernel vs flashinfer trtllm-gen paged decode (same bytes):
# timing, launch configuration and DRAM bytes per launch, one full ncu capture of each
cd "$(dirname "$0")/.."
O=gpurun_out/r2ad; mkdir -p $O
timeout 300 python tools/decode_vs_trtllm.py --time --launches 1 > $O/time.json 2> $O/time.err; echo "time rc=$?" >> $O/status
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,launch__registers_per_thread,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__cluster_dim_x
timeout 600 ncu --nvtx --nvtx-include "cmp/" --metrics $M --clock-control none --csv --log-file $O/launches.csv python tools/decode_vs_trtllm.py --launches 3 > $O/launches.log 2>&1; echo "launches rc=$?" >> $O/status
timeout 900 ncu --nvtx --nvtx-include "cmp/" --set full --clock-control none -c 2 -o $O/full python tools/decode_vs_trtllm.py --launches 1 > $O/full.log 2>&1; echo "full rc=$?" >> $O/status
cat $O/status $O/time.json
