"""Write profiles/decode_traffic.json — roofline.traffic per bench config —
from `ncu --set full` captures of ONE decode launch inside `bench.py
--profile-steps` for each config (tools/gpu_r2j.sh; late r02 recapture: tools/gpu_r2be.sh).

    python tools/make_traffic.py gpurun_out/r2j > profiles/decode_traffic.json

Keys are `<config>/<path>`, the key bench.py looks up. The growth trace has no
entry: its launches sweep 256..32,752 tokens, so no single capture stands for
them (bench reports traffic = null there).
"""

import glob
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main(d: str) -> None:
    out = {"note": ("dram__bytes_read.sum + dram__bytes_write.sum of one decode launch, from an "
                    "`ncu --set full --clock-control none` capture inside `bench.py --config C "
                    "--profile-steps 3` (tools/gpu_r2j.sh; late r02 recapture: tools/gpu_r2be.sh); one launch = one layer of the config's "
                    "batch at its context")}
    for rep in sorted(glob.glob(os.path.join(d, "decode_*.ncu-rep"))):
        key = os.path.basename(rep)[len("decode_"):-len(".ncu-rep")].replace("__", "/")
        s = json.loads(subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), rep],
                                      capture_output=True, text=True, check=True).stdout)
        out[key] = {"kernel": s.get("kernel"), "dram_bytes_per_launch": int(s["dram_traffic_bytes"]),
                    "duration_us": round(s["duration"] * 1e6, 2),
                    "source": f"profiles/r02/ncu_late/{os.path.basename(rep)[:-8]}.json"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
