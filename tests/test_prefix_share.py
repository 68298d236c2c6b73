"""Cross-device prefix sharing: host logic on CPU.

The GPU half (export/import through the driver, one and two processes) is
tests/test_prefix_share_gpu.py.
"""

import pytest

import paper_2407_15309_b200 as vt
from paper_2407_15309_b200.prefix_share import SharedPrefix, import_prefix
from paper_2407_15309_b200.vmm import PhysicalHandle

MIB = 1 << 20


def _stack():
    cfg = vt.SimConfig(capacity_bytes=64 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(32, 8, 128, 2), max_seq_len=1024,
                       initial_alloc_tokens=0)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes))
    ops = vt.VTensorOps(dev, vt.TensorPool(cfg.tokens_per_chunk), cfg)
    return cfg, dev, ops, vt.VTensorScheduler(ops)


def test_imported_chunk_is_never_parked_for_reuse():
    pool = vt.TensorPool(16)
    local, imported = PhysicalHandle(1), PhysicalHandle(2, imported=True)
    for h in (local, imported):
        pool.add_entry(h)
        pool.incref(h, 7)
    pool.decref(local, 7)
    pool.decref(imported, 7)
    assert pool.free_handles() == [local]          # the lazy free list: local memory only
    assert pool.released_imports == [imported]     # another pool's memory: handed back
    assert pool.take_free(2) == [local]


def test_vto_drops_released_imports():
    """unmap_space decrefs; an imported chunk that nobody maps any more is
    dropped from the pool and its device reference destroyed."""
    cfg, dev, ops, sched = _stack()
    space = ops.v_alloc(cfg.max_seq_len)
    h = dev.create_chunk()           # stands in for an imported handle on the simulated device
    h.imported = True
    ops.pool.add_entry(h)
    local = ops.p_alloc(1)
    ops.map_chunks(space, [h] + local)
    assert ops.pool.entries[h.id].referrers == {space.space_id}
    ops.unmap_space(space)
    assert h.id not in ops.pool.entries
    assert h.id not in {x.id for x in dev.live_handles()}
    assert ops.pool.free_handles() == local     # the local chunk parks as usual


def test_simulated_device_refuses_export_and_import():
    cfg, dev, ops, sched = _stack()
    h = dev.create_chunk()
    with pytest.raises(ValueError):
        dev.export_chunk(h)
    with pytest.raises(ValueError):
        dev.import_chunk(0)


def test_import_prefix_rejects_geometry_mismatch():
    cfg, dev, ops, sched = _stack()
    bad = SharedPrefix(matched_tokens=32, fds=[], tokens_per_chunk=32, chunk_bytes=cfg.chunk_size_bytes)
    with pytest.raises(ValueError):
        import_prefix(sched, "r", list(range(64)), bad)
