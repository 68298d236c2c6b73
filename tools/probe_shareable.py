"""Probe: idle cost of cuMemCreate / cuMemMap+SetAccess for ordinary vs
shareable (POSIX-fd exportable) chunks. python tools/probe_shareable.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_15309_b200 as vt  # noqa: E402

MIB = 1 << 20
out = {}
for shareable in (False, True, False, True):
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(2048 * 2 * MIB, 2 * MIB), cuda_ordinal=0)
    if shareable:
        dev.set_shareable(True)
    rng = dev.reserve_address(256 * 2 * MIB)
    hs = [dev.create_chunk() for _ in range(256)]
    dev.wait()
    for i in range(0, 256, 4):
        dev.map_pages(rng, i, hs[i:i + 4])
    dev.wait()
    s = dev.driver_stats()
    key = "shareable" if shareable else "plain"
    out.setdefault(key, []).append({
        "create_us": round(s["create_ns_total"] / s["create_calls"] / 1e3, 1),
        "map_us": round(s["map_ns_total"] / s["map_calls"] / 1e3, 1),
        "access_us_per_4": round(s["access_ns_total"] / s["access_calls"] / 1e3, 1)})
    dev.close()
print(json.dumps(out))
