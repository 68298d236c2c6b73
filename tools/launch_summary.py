"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean device time, and share of the total.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN/launches_bench.json
"""

import csv
import json
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.match(r"(?:void )?([\w:]+(?:<[^<>]*>)?)", name)
    return m.group(1) if m else name[:60]


def main(path: str) -> None:
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    total = sum(t for _, t in agg.values())
    ours = {k: v for k, v in agg.items() if k.startswith(("vt::", "decode", "prefill", "kv_append", "vt"))
            or "anonymous" in k}
    out = {
        "source": path,
        "note": "ncu launch list: cold-cache, serialised replay; compare shares, not absolutes",
        "kernels": {k: {"launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 2),
                        "share": round(t / total, 4)}
                    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])},
        "total_us": round(total, 1),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
