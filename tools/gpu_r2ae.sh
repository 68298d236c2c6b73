#!/bin/bash
# round 2: decode KV tensor-map L2 promotion (none / 64B / 128B / 256B) vs trtllm-gen
cd "$(dirname "$0")/.."
O=gpurun_out/r2ae; mkdir -p $O
for p in 3 2 0 1 3 2; do
  VT_TMAP_PROMO=$p timeout 300 python tools/decode_vs_trtllm.py --time --launches 1 >> $O/time_p$p.json 2>> $O/time.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_ltcfabric.sum
for p in 3 2 0; do
VT_TMAP_PROMO=$p timeout 600 ncu --nvtx --nvtx-include "cmp/" --metrics $M --clock-control none --csv --log-file $O/l2_p$p.csv python tools/decode_vs_trtllm.py --launches 2 > /dev/null 2>&1
done
for p in 3 2 0 1; do echo "promo $p"; cat $O/time_p$p.json; done
