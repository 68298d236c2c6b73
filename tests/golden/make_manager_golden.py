"""Generate tests/golden/manager_streams.json from the REFERENCE kvsim.

Runs every stream in tests/manager_streams.STREAMS through the unmodified
reference package at /root/reference/pkg/src (read-only, imported, never
copied) and records the digest of the canonical manager dump after every op,
the per-op events, and the full final dump. The GPU box has no
/root/reference, so these committed vectors are what the CUDA-backend parity
tests check against.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_manager_golden.py
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import kvsim  # noqa: E402  (the reference)
import manager_streams as ms  # noqa: E402


def main() -> None:
    assert kvsim.__file__.startswith("/root/reference"), kvsim.__file__
    cfgs = ms.stream_configs(kvsim)
    out = {"generator": "reference kvsim @ /root/reference/pkg/src", "streams": []}
    for name, seed, steps in ms.STREAMS:
        digests = []
        st, events = ms.run_stream(kvsim, cfgs[name], seed, steps,
                                   on_step=lambda i, s: digests.append(ms.digest(ms.dump(s))))
        final = ms.dump(st)
        out["streams"].append({
            "config": name, "seed": seed, "steps": steps,
            "digests": digests, "events": events,
            "final_log_len": len(final["log"]),
            "final_digest": ms.digest(final),
            "call_mix": {op: sum(1 for c in final["log"] if c[1] == op)
                         for op in sorted({c[1] for c in final["log"]})},
        })
        print(name, seed, steps, "calls", len(final["log"]), out["streams"][-1]["call_mix"])
    with open(os.path.join(HERE, "manager_streams.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
