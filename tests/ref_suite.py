"""Run the reference's own test suite against this package (drop-in proof).

Builds a throw-away ``kvsim`` package in a temp dir whose L0-L3 modules
(config, device, pool, ops, scheduler) re-export THIS package's
implementation, while the out-of-scope modules (engine, metrics, trace,
verify, baselines, cli, __init__) are symlinks to the read-only reference at
/root/reference/pkg/src/kvsim. Nothing from the reference is copied into the
repo. Then runs ``pytest /root/reference/pkg/tests`` against it.

Usage: python tests/ref_suite.py [--cuda ORDINAL] [pytest args...]
With --cuda the shim's CUDA-driver backend is used wherever a test builds a
device with 2 MiB chunks (tiny-chunk tests stay simulated: the driver cannot
map 128-byte pages).
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

REF_PKG = "/root/reference/pkg"
REF_SRC = os.path.join(REF_PKG, "src", "kvsim")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHIMS = {
    "config.py": (
        "from paper_2407_15309_b200.geometry import GIB, KIB, MIB, ModelGeometry, SimConfig\n"
        # CLI size parsing is out of scope: the reference's own
        "import importlib.util as _u\n"
        "_s = _u.spec_from_file_location('_kvsim_ref_config', {ref_config!r})\n"
        "_m = _u.module_from_spec(_s)\n"
        "import sys as _sys\n"
        "_sys.modules['_kvsim_ref_config'] = _m\n"
        "_s.loader.exec_module(_m)\n"
        "parse_size, format_size = _m.parse_size, _m.format_size\n"
    ),
    "device.py": (
        "from paper_2407_15309_b200.vmm import (ChunkStillMapped, DeviceCall, DeviceConfig, "
        "DeviceError, DeviceOutOfMemory, DeviceStats, IndexOutOfRange, InvalidSize, "
        "PageAlreadyMapped, PageNotMapped, PhysicalHandle, RangeStillMapped, StaleHandle, "
        "UnknownRange, VirtualRange)\n"
        "from paper_2407_15309_b200.vmm import VirtualMemoryDevice as _Dev\n"
        "import os as _os\n"
        "_ORD = _os.environ.get('VT_REF_SUITE_CUDA')\n"
        "class VirtualMemoryDevice(_Dev):\n"
        "    def __init__(self, config, cuda_ordinal=None):\n"
        "        if cuda_ordinal is None and _ORD is not None and config.chunk_size_bytes % (2 << 20) == 0:\n"
        "            cuda_ordinal = int(_ORD)\n"
        "        super().__init__(config, cuda_ordinal)\n"
    ),
    "pool.py": (
        "from paper_2407_15309_b200.tensor_pool import (ChunkState, PhysicalEntry, "
        "PoolStateError, PrefixTree, RadixNode, SpaceState, TensorPool, UnknownReferrer, "
        "VirtualSpace, VirtualTensor)\n"
    ),
    "ops.py": (
        "from paper_2407_15309_b200.vto import CapacityExceeded, OpRecord, ReclaimReport, "
        "VTensorOps\n"
    ),
    "scheduler.py": (
        "from paper_2407_15309_b200.vts import AdmitStats, ExceedsMaxSeqLen, RequestMem, "
        "VTensorScheduler\n"
    ),
}
LINKED = ("__init__.py", "engine.py", "metrics.py", "trace.py", "verify.py", "baselines.py",
          "cli.py")


def kvsim_source() -> str | None:
    """The reference kvsim sources: /root/reference here, else the unmodified
    install under baseline/_ref (it travels to the GPU box with the repo)."""
    for d in (REF_SRC, os.path.join(REPO, "baseline", "_ref", "kvsim")):
        if os.path.isfile(os.path.join(d, "engine.py")):
            return d
    return None


def build_kvsim_overlay(root: str, src: str | None = None) -> str:
    src = src or REF_SRC
    pkg = os.path.join(root, "kvsim")
    os.makedirs(pkg, exist_ok=True)
    for name, body in SHIMS.items():
        with open(os.path.join(pkg, name), "w") as f:
            f.write(body.replace("{ref_config!r}", repr(os.path.join(src, "config.py"))))
    for name in LINKED:
        os.symlink(os.path.join(src, name), os.path.join(pkg, name))
    return root


def main(argv: list[str]) -> int:
    env = dict(os.environ)
    if argv[:1] == ["--cuda"]:
        env["VT_REF_SUITE_CUDA"] = argv[1]
        argv = argv[2:]
    with tempfile.TemporaryDirectory() as tmp:
        build_kvsim_overlay(tmp)
        env["PYTHONPATH"] = os.pathsep.join([tmp, REPO, env.get("PYTHONPATH", "")])
        env["PYTHONDONTWRITEBYTECODE"] = "1"
        cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-q",
               "--rootdir", tmp, os.path.join(REF_PKG, "tests"), *argv]
        return subprocess.call(cmd, env=env, cwd=tmp)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
