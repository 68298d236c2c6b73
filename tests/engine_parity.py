"""Run the REFERENCE ServingEngine on a few traces and print CSV + summary.

  mode=reference : kvsim from /root/reference (allocator = its VTensorAdapter)
  mode=ours      : kvsim overlay (tests/ref_suite.py) whose L0-L3 are this
                   package AND whose vtensor allocator is this package's
                   VTensorAdapter (paper_2407_15309_b200.adapter)
Used by tests/test_adapter.py (the two outputs must be byte-identical).
"""

import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))


def main(mode: str) -> None:
    if mode == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
    else:
        sys.path.insert(0, os.path.dirname(HERE))
        sys.path.insert(0, HERE)
        from ref_suite import build_kvsim_overlay

        sys.path.insert(0, build_kvsim_overlay(tempfile.mkdtemp()))
    import kvsim
    import kvsim.engine as eng

    if mode == "ours":
        from paper_2407_15309_b200.adapter import VTensorAdapter

        orig = eng.build_allocator
        eng.build_allocator = lambda name, dev, cfg: (VTensorAdapter(dev, cfg) if name == "vtensor"
                                                      else orig(name, dev, cfg))
    GIB = 1 << 30
    runs = {
        "prefix_share": (kvsim.SimConfig(max_seq_len=16384),
                         kvsim.generate_trace("prefix_share", seed=5, requests=8)),
        "multi_turn": (kvsim.SimConfig(max_seq_len=12288),
                       kvsim.generate_trace("multi_turn", seed=7, conversations=3, turns=2)),
        "reduced_preempt": (kvsim.SimConfig(capacity_bytes=13 * GIB, weights_bytes=12 * GIB,
                                            max_seq_len=12288, max_batch=4),
                            kvsim.generate_trace("single_gen", seed=3, requests=4)),
    }
    out = {}
    for name, (cfg, trace) in runs.items():
        rep = eng.run_trace(trace, cfg)
        out[name] = {"csv": rep.to_csv(), "summary": rep.summary(),
                     "admissions": rep.admissions, "stalls": rep.stall_count,
                     "preemptions": rep.preemption_count}
    print(json.dumps(out, sort_keys=True, default=str))


if __name__ == "__main__":
    main(sys.argv[1])
