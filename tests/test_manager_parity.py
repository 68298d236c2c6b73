"""Manager (L0-L3) parity: bit-exact against the reference kvsim.

* golden: per-op digests of the canonical state dump recorded from the
  reference (tests/golden/make_manager_golden.py) — replayed on the simulated
  shim here and on the CUDA-driver shim on the GPU box;
* lock-step: the live reference and this package driven side by side, full
  dump compared after every op (CPU container only: needs /root/reference);
* the reference's own 154-test suite against this package (tests/ref_suite.py).
"""

import json
import os
import subprocess
import sys

import pytest

import manager_streams as ms
import paper_2407_15309_b200 as vt
from conftest import HAVE_REFERENCE, REFERENCE_SRC, TESTS

GOLDEN = json.load(open(os.path.join(TESTS, "golden", "manager_streams.json")))


def _replay(stream, device_kwargs=None, fence=None):
    cfgs = ms.stream_configs(vt)
    digests = []

    def on_step(i, st):
        if st.dev.is_cuda:
            st.dev.wait()  # driver half must have landed; state is already synchronous
        digests.append(ms.digest(ms.dump(st)))

    st, events = ms.run_stream(vt, cfgs[stream["config"]], stream["seed"], stream["steps"],
                               on_step=on_step, device_kwargs=device_kwargs, fence=fence)
    return st, digests, events


@pytest.mark.parametrize("idx", range(len(GOLDEN["streams"])))
def test_streams_match_reference_golden(idx):
    stream = GOLDEN["streams"][idx]
    st, digests, events = _replay(stream)
    assert json.loads(json.dumps(events)) == stream["events"]
    first_bad = next((i for i, (a, b) in enumerate(zip(digests, stream["digests"])) if a != b),
                     None)
    assert first_bad is None, f"state diverged from reference after op {first_bad}"
    assert len(digests) == len(stream["digests"])


@pytest.mark.skipif(not HAVE_REFERENCE, reason="reference kvsim not present")
@pytest.mark.parametrize("name,seed,steps", [("toy", 11, 150), ("llama8b", 12, 150),
                                             ("llama70b_g16_h2", 13, 150)])
def test_lockstep_full_dump_against_live_reference(name, seed, steps):
    sys.path.insert(0, REFERENCE_SRC)
    try:
        import kvsim
    finally:
        sys.path.remove(REFERENCE_SRC)
    ref_dumps, our_dumps = [], []
    ms.run_stream(kvsim, ms.stream_configs(kvsim)[name], seed, steps,
                  on_step=lambda i, s: ref_dumps.append(ms.dump(s)))
    ms.run_stream(vt, ms.stream_configs(vt)[name], seed, steps,
                  on_step=lambda i, s: our_dumps.append(ms.dump(s)))
    assert len(ref_dumps) == len(our_dumps)
    for i, (a, b) in enumerate(zip(ref_dumps, our_dumps)):
        assert a == b, f"op {i}: " + ", ".join(k for k in a if a[k] != b[k])


@pytest.mark.skipif(not HAVE_REFERENCE, reason="reference kvsim not present")
def test_reference_suite_passes_against_this_package():
    """All 154 reference tests, with kvsim's L0-L3 swapped for this package."""
    r = subprocess.run([sys.executable, os.path.join(TESTS, "ref_suite.py"), "-x"],
                       capture_output=True, text=True, timeout=600)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "154 passed" in tail, tail


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(GOLDEN["streams"])))
def test_streams_match_reference_golden_on_cuda_driver(cuda_ok, idx):
    """Same op streams with real cuMemCreate/cuMemMap on the B200: identical
    manager state, and the driver really executed every map/unmap."""
    import torch

    stream = GOLDEN["streams"][idx]
    torch.cuda.init()
    s = torch.cuda.current_stream().cuda_stream
    st, digests, events = _replay(stream, device_kwargs={"cuda_ordinal": 0},
                                  fence=lambda st: st.dev.fence(s))
    st.dev.wait()
    assert digests == stream["digests"]
    d = st.dev.driver_stats()
    mix = stream["call_mix"]
    assert d["map_calls"] == mix["map_page"]
    assert d["unmap_calls"] == mix["unmap_page"]
    assert d["create_calls"] == mix["create_chunk"]
    assert d["destroy_calls"] == mix["destroy_chunk"]
    st.dev.close()
