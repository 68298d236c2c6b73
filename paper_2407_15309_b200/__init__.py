"""B200-native vTensor: VMM-backed KV cache manager + sm_100a attention kernels.

The manager half keeps the Python API of the reference package ``kvsim``
(names below mirror kvsim/__init__.py:75-145 for layers L0-L3 and the geometry
config) on top of ``libvtensor.so``, a C-ABI shim over the CUDA driver VMM.
The attention half (decode split-KV, tcgen05 prefill, KV append) lives in
``libvtattn.so`` and is reached through :mod:`paper_2407_15309_b200.attention`.
"""

from .geometry import GIB, KIB, MIB, ModelGeometry, SimConfig
from .vmm import (
    ChunkStillMapped,
    DeviceCall,
    DeviceConfig,
    DeviceError,
    DeviceOutOfMemory,
    DeviceStats,
    DriverFailure,
    IndexOutOfRange,
    InvalidSize,
    PageAlreadyMapped,
    PageNotMapped,
    PhysicalHandle,
    RangeStillMapped,
    StaleHandle,
    UnknownRange,
    VirtualMemoryDevice,
    VirtualRange,
)
from .tensor_pool import (
    ChunkState,
    PhysicalEntry,
    PoolStateError,
    PrefixTree,
    RadixNode,
    SpaceState,
    TensorPool,
    UnknownReferrer,
    VirtualSpace,
    VirtualTensor,
)
from .vto import CapacityExceeded, OpRecord, ReclaimReport, VTensorOps
from .vts import AdmitStats, ExceedsMaxSeqLen, RequestMem, VTensorScheduler

__version__ = "0.1.0"

__all__ = [
    "GIB", "KIB", "MIB", "ModelGeometry", "SimConfig",
    "ChunkStillMapped", "DeviceCall", "DeviceConfig", "DeviceError", "DeviceOutOfMemory",
    "DeviceStats", "DriverFailure", "IndexOutOfRange", "InvalidSize", "PageAlreadyMapped",
    "PageNotMapped", "PhysicalHandle", "RangeStillMapped", "StaleHandle", "UnknownRange",
    "VirtualMemoryDevice", "VirtualRange",
    "ChunkState", "PhysicalEntry", "PoolStateError", "PrefixTree", "RadixNode", "SpaceState",
    "TensorPool", "UnknownReferrer", "VirtualSpace", "VirtualTensor",
    "CapacityExceeded", "OpRecord", "ReclaimReport", "VTensorOps",
    "AdmitStats", "ExceedsMaxSeqLen", "RequestMem", "VTensorScheduler",
]
