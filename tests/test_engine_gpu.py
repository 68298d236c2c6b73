"""SURVEY.md §8(f) row 1 and SURVEY §7.2 item 4 on the B200: the reference's
unmodified ServingEngine (kvsim/engine.py:322-583) runs traces with this
package under it (CUDA-driver VMM device, GpuServingAdapter) and the real
attention kernels in its compute slot (engine.py:499-511):

* the engine report — per-step CSV, summary, admissions, preemptions — is
  byte-identical to the reference's own CPU run of the same trace (manager
  parity with kernels reading the pages);
* attention outputs match the CPU oracle through a K/V mirror (every step for
  the config-1 toy trace, 3,840 steps; sampled steps for the long traces) and
  the cache bytes read back through the request VAs equal the mirror;
* the driver executed exactly the logged VMM calls; the memory lane (host
  waits for mappings, GPU idle behind them) is measured.

The engine source is the reference's (kvsim); on the GPU box it comes from
the unmodified install under baseline/_ref.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO, TESTS

sys.path.insert(0, TESTS)
from ref_suite import kvsim_source  # noqa: E402

RUN = os.path.join(TESTS, "engine_gpu_run.py")


def _run(mode, trace, *extra, timeout=1800):
    proc = subprocess.run([sys.executable, RUN, mode, trace, *extra], capture_output=True,
                          text=True, timeout=timeout, cwd=REPO)
    assert proc.returncode == 0, proc.stderr[-4000:]
    return json.loads(proc.stdout.strip().splitlines()[-1])


TRACES = {
    # trace: (check_every, expected preemptions > 0)
    "toy_cfg1": (1, False),
    "multi_turn": (64, False),
    "reduced_preempt": (64, True),
}


@pytest.mark.gpu
@pytest.mark.parametrize("trace", list(TRACES))
def test_reference_engine_with_gpu_compute(cuda_ok, trace):
    if kvsim_source() is None:
        pytest.skip("reference engine source not present (neither /root/reference nor baseline/_ref)")
    every, preempts = TRACES[trace]
    ref = _run("reference", trace)
    got = _run("gpu", trace, "--check-every", str(every))
    for key in ("csv", "summary", "admissions", "stalls", "preemptions"):
        assert got[key] == ref[key], f"{trace}: engine {key} differs from the reference run"
    g = got["gpu"]
    c = g["check"]
    assert not c["fail"], c["fail"]
    assert c["max_rel_err"] <= 2e-2
    assert c["prefill_checks"] > 0 and c["decode_checks"] > 0 and c["byte_checks"] > 0
    if trace == "toy_cfg1":
        assert g["steps"] == 3840 and c["decode_checks"] == 3839  # step 0 is the prefill
        assert g["logged_calls"] == {"reserve_address": 8, "create_chunk": 45, "map_page": 64,
                                     "unmap_page": 64, "destroy_chunk": 45,
                                     "release_address": 8}, g["logged_calls"]
    if preempts:
        assert got["preemptions"] > 0
    d = g["driver"]
    lc = g["logged_calls"]
    assert d["map_calls"] == lc.get("map_page", 0)
    assert d["unmap_calls"] == lc.get("unmap_page", 0)
    assert d["create_calls"] + d["reserve_hits"] >= lc.get("create_chunk", 0)
