"""Row a25: the reference's own ServingEngine, driving this package's
VTensorAdapter over this package's manager, produces byte-identical CSV
reports, summaries and admission records to the pure reference (prefix-share
frugality, multi-turn records, preemption under memory pressure)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import HAVE_REFERENCE, TESTS


@pytest.mark.skipif(not HAVE_REFERENCE, reason="reference kvsim not present")
def test_reference_engine_with_our_adapter_is_identical():
    outs = {}
    for mode in ("reference", "ours"):
        r = subprocess.run([sys.executable, os.path.join(TESTS, "engine_parity.py"), mode],
                           capture_output=True, text=True, timeout=600,
                           env={**os.environ, "PYTHONDONTWRITEBYTECODE": "1"})
        assert r.returncode == 0, r.stderr[-3000:]
        outs[mode] = json.loads(r.stdout)
    ref, ours = outs["reference"], outs["ours"]
    assert ref.keys() == ours.keys()
    for name in ref:
        assert ours[name]["csv"] == ref[name]["csv"], name
        assert ours[name]["summary"] == ref[name]["summary"], name
        assert ours[name]["admissions"] == ref[name]["admissions"], name
    assert ref["reduced_preempt"]["preemptions"] > 0
    assert ref["prefix_share"]["summary"]["pinned_chunks"] == 500 + 7 * 125


def test_adapter_protocol_surface():
    from paper_2407_15309_b200.adapter import VTensorAdapter

    for m in ("startup", "can_admit", "admit", "prefill_reserve", "ensure_capacity",
              "mark_prefilled", "append_token", "finish", "release", "shutdown", "kv_stats",
              "extra_summary"):
        assert callable(getattr(VTensorAdapter, m))
