"""bench.py's driver contract on the CPU side: the reference arm (the CPU
restatement of the path, timed on the host cores) prints one JSON line with
the keys the driver reads, on the same metric / unit as our arm."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO


def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    proc = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "1"],
                          capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "decode-attn KV GB/s (% of HBM peak) and tokens/s; vTensor extend latency"
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    ext = d["extend"]
    assert ext["extend_1chunk_us_p50"] > 0 and ext["prefix_match_2048_512_us_p50"] > 0


@pytest.mark.gpu
def test_our_arm_prints_the_contract_line(cuda_ok):
    proc = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--steps", "3",
                           "--warmup", "3", "--no-prefill", "--no-qkv", "--no-cpu-baseline"],
                          capture_output=True, text=True, timeout=900, cwd=REPO)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks", "extend"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"].startswith("llama3-8b-decode")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert d["gpu_launches"] >= 33 * 3  # KV append + 32 decode layers per step
    assert d["extend"]["gpu_stalled_steps"] == 0
