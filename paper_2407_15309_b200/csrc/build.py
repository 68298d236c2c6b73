"""In-tree build of the native libraries (no JIT cache: the .so files travel
to the GPU box with the repo snapshot).

  libvtensor.so : g++ -O2, C++17, dlopens libcuda at run time (include/vtensor.h)
  _vtfast*.so   : gcc -O2, CPython entry points for the manager's per-token
                  calls into libvtensor.so (symbols resolved from the
                  RTLD_GLOBAL-loaded shim, so an A/B shim build is honoured)
  libvtattn.so  : nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo
                  (include/vt_attention.h)
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

CSRC = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(CSRC)
REPO = os.path.dirname(PKG)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    hdrs = glob.glob(os.path.join(REPO, "include", "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    shim_src = [os.path.join(CSRC, "vtensor_shim.cpp")]
    shim = os.path.join(PKG, "libvtensor.so")
    if force or _stale(shim, shim_src + hdrs):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-Wall", f"-I{CUDA}/include",
              "-o", shim, *shim_src, "-ldl", "-lpthread"])
    import sysconfig

    fast_src = [os.path.join(CSRC, "vt_pyfast.c")]
    fast = os.path.join(PKG, "_vtfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or _stale(fast, fast_src + hdrs):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-Wall", f"-I{sysconfig.get_paths()['include']}",
              "-o", fast, *fast_src])
    cu_src = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    attn = os.path.join(PKG, "libvtattn.so")
    if force or _stale(attn, cu_src + hdrs):
        extra = ["-Xptxas", "-v"] if verbose_ptxas else []
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC", "-shared", *extra, "-o", attn, *cu_src])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
