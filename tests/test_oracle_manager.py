"""Pin the manager oracle (oracle/vtm_ref.py) to the reference: every golden
stream recorded from kvsim itself must replay to identical per-op digests."""

import json
import os

import pytest

import manager_streams as ms
from conftest import TESTS
from oracle import vtm_ref

GOLDEN = json.load(open(os.path.join(TESTS, "golden", "manager_streams.json")))


@pytest.mark.parametrize("idx", range(len(GOLDEN["streams"])))
def test_oracle_replays_reference_golden(idx):
    stream = GOLDEN["streams"][idx]
    digests = []
    st, events = ms.run_stream(vtm_ref, ms.stream_configs(vtm_ref)[stream["config"]],
                               stream["seed"], stream["steps"],
                               on_step=lambda i, s: digests.append(ms.digest(ms.dump(s))))
    assert json.loads(json.dumps(events)) == stream["events"]
    bad = next((i for i, (a, b) in enumerate(zip(digests, stream["digests"])) if a != b), None)
    assert bad is None, f"oracle diverged from the reference after op {bad}"
