"""Summarise an ncu report into the numbers bench.py and DESIGN.md cite.

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [--bytes N | --flops N] > profiles/x.json

Reads the raw page (CSV) with `ncu -i`, extracts duration, DRAM traffic,
DRAM/tensor/issue utilisation and the top stall reasons, and (given the
algorithmic bytes or FLOPs of the launch) the achieved GB/s or TFLOP/s.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_ncu_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}

SCALE = {"usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0,
         "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--bytes", type=float, default=0.0)
    ap.add_argument("--flops", type=float, default=0.0)
    ap.add_argument("--name", default="")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out: dict = {"report": args.report, "kernel": vals[hdr.index("Kernel Name")]
                 if "Kernel Name" in hdr else args.name}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[i], 1.0)
            except ValueError:
                continue
            out[name] = x
    stalls = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                stalls.append((h.split("stalled_")[-1], float(vals[i])))
            except ValueError:
                pass
    tot = sum(v for _, v in stalls) or 1.0
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                             for k, v in sorted(stalls, key=lambda x: -x[1])[:6]}
    dur = out.get("duration")
    if dur:
        traffic = out.get("dram_read", 0.0) + out.get("dram_write", 0.0)
        out["dram_traffic_bytes"] = traffic
        out["dram_GBps"] = traffic / dur / 1e9
        if args.bytes:
            out["algorithmic_bytes"] = args.bytes
            out["achieved_GBps"] = args.bytes / dur / 1e9
            out["traffic_over_algorithmic"] = traffic / args.bytes
        if args.flops:
            out["algorithmic_flops"] = args.flops
            out["achieved_TFLOPs"] = args.flops / dur / 1e12
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
