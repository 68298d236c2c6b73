"""Cross-device prefix sharing on the B200.

Two managers stand for two GPUs' pools (one GPU in this environment; on a
multi-GPU box the borrower would open cuda_ordinal=1 and the same mapping's
cuMemSetAccess would grant peer access over NVLink). The donor records a
conversation; the borrower imports the matched chunks by their exported
handles, maps them by identity into its own VA and runs the prefix-prefill
kernel over them in place. Checked: bytes identical through both VAs, a write
through the donor's VA is visible to the borrower (same physical memory, not
a copy), attention matches the oracle, the borrower's budget excludes the
imported chunks and releasing the borrower leaves the donor's state intact.
"""

import multiprocessing as mp
import socket

import pytest
import torch

from oracle.attention_ref import prefill_attention_ref, rel_err
from paper_2407_15309_b200.attention import kv_tensor_maps, prefill_attention
from paper_2407_15309_b200.kv_layout import chunk_view, read_kv
from paper_2407_15309_b200.prefix_share import (export_prefix, import_prefix,
                                                recv_shared_prefix, send_shared_prefix)
from vt_gpu_util import cuda_stack

PREFIX, NEW = 1024, 256


def _donor(seed=0):
    st = cuda_stack(32, 8, 32, 4096, capacity_chunks=512)
    st.dev.set_shareable(True)
    base = [(i * 13 + 1) % 501 for i in range(PREFIX)]
    st.sched.create("conv", base)
    st.sched.mark_prefilled("conv")
    st.dev.wait()
    va = st.dev.va(st.sched.mem["conv"].vt.space.rng)
    v = chunk_view(va, PREFIX // st.cfg.tokens_per_chunk, st.geo)
    v.copy_(torch.randn(v.shape, generator=torch.Generator(device="cuda").manual_seed(seed),
                        device="cuda").to(torch.bfloat16))
    torch.cuda.synchronize()
    assert st.sched.prefix_record("conv")
    return st, base, va


@pytest.mark.gpu
def test_prefix_shared_across_managers(cuda_ok):
    donor, base, dva = _donor()
    borrower = cuda_stack(32, 8, 32, 4096, capacity_chunks=512)
    tpc = borrower.cfg.tokens_per_chunk
    tokens = base + [7000 + k for k in range(NEW)]
    donor_entries = {hid: set(e.referrers) for hid, e in donor.pool.entries.items()}

    shared = export_prefix(donor.sched, tokens)
    assert shared.matched_tokens == PREFIX and len(shared.fds) == PREFIX // tpc
    rm, stats = import_prefix(borrower.sched, "turn", tokens, shared)
    assert stats.identity_ok and stats.shared_tokens == PREFIX
    assert stats.chunks_created == NEW // tpc
    # imported chunks live in the donor's budget, not the borrower's
    assert borrower.dev.created_bytes == (NEW // tpc) * borrower.cfg.chunk_size_bytes
    borrower.dev.wait()
    bva = borrower.dev.va(rm.vt.space.rng)
    assert bva != dva

    for layer in (0, 31):
        k_d, v_d = read_kv(dva, PREFIX, layer, donor.geo)
        k_b, v_b = read_kv(bva, PREFIX, layer, borrower.geo)
        assert torch.equal(k_d, k_b) and torch.equal(v_d, v_b)
    chunk_view(dva, 1, donor.geo)[0, 5, 1, 3].fill_(2.5)  # hard link, not a copy
    torch.cuda.synchronize()
    assert torch.all(chunk_view(bva, 1, borrower.geo)[0, 5, 1, 3] == 2.5)

    # the new turn's own KV, then prefill over shared prefix + new tokens
    own = chunk_view(bva, (PREFIX + NEW) // tpc, borrower.geo)[PREFIX // tpc:]
    own.copy_(torch.randn(own.shape, device="cuda").to(torch.bfloat16))
    q = torch.randn(1, NEW, 32, 128, device="cuda").to(torch.bfloat16)
    maps = kv_tensor_maps([bva], [PREFIX + NEW], borrower.geo)
    out = prefill_attention(q, maps, torch.tensor([PREFIX], dtype=torch.int32, device="cuda"), 9,
                            borrower.geo)
    torch.cuda.synchronize()
    k, v = read_kv(bva, PREFIX + NEW, 9, borrower.geo)
    ref = prefill_attention_ref(q[0].cpu(), k.cpu(), v.cpu(), PREFIX)
    assert rel_err(out[0].cpu(), ref) <= 2e-2

    # release: the borrower drops its references; the donor is untouched
    k_before = read_kv(dva, PREFIX, 0, donor.geo)[0]
    borrower.sched.mark_prefilled("turn")
    borrower.sched.release("turn")
    borrower.dev.wait()
    assert not any(h.imported for h in borrower.dev.live_handles())
    assert not borrower.pool.released_imports
    assert {hid: set(e.referrers) for hid, e in donor.pool.entries.items()} == donor_entries
    assert torch.equal(read_kv(dva, PREFIX, 0, donor.geo)[0], k_before)


def _borrower_proc(sock, result_q):
    """Another process (another rank): receive the fds, import, map, checksum."""
    torch.cuda.init()
    try:
        st = cuda_stack(32, 8, 32, 4096, capacity_chunks=512)
        shared = recv_shared_prefix(sock)
        tokens = [(i * 13 + 1) % 501 for i in range(PREFIX)] + [1] * NEW
        rm, stats = import_prefix(st.sched, "remote", tokens, shared)
        st.dev.wait()
        k, v = read_kv(st.dev.va(rm.vt.space.rng), PREFIX, 3, st.geo)
        result_q.put((stats.identity_ok, float(k.float().sum()), float(v.float().abs().sum())))
        st.sched.release("remote")
        st.dev.wait()
    except Exception as exc:  # surfaced by the parent
        result_q.put(repr(exc))


@pytest.mark.gpu
def test_prefix_shared_across_processes(cuda_ok):
    donor, base, dva = _donor(seed=4)
    parent, child = socket.socketpair(socket.AF_UNIX, socket.SOCK_STREAM)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_borrower_proc, args=(child, q))
    p.start()
    shared = export_prefix(donor.sched, base + [1] * NEW)
    send_shared_prefix(parent, shared)
    res = q.get(timeout=240)
    p.join(timeout=60)
    assert not isinstance(res, str), res
    identity_ok, ksum, vabs = res
    k, v = read_kv(dva, PREFIX, 3, donor.geo)
    assert identity_ok
    assert ksum == float(k.float().sum()) and vabs == float(v.float().abs().sum())
    assert p.exitcode == 0


@pytest.mark.gpu
def test_prefix_shared_across_gpus(cuda_ok):
    """the donor's pool on GPU 0, the borrower's on GPU 1.
    The imported chunks stay in GPU 0's HBM; the borrower's cuMemSetAccess
    grants GPU 1 access to them (peer over NVLink), and GPU 1's prefill kernel
    reads the shared prefix in place through the borrower's VA."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (the driver's multi-GPU box)")
    with torch.cuda.device(0):
        donor, base, dva = _donor(seed=7)
        tokens = base + [9000 + k for k in range(NEW)]
        shared = export_prefix(donor.sched, tokens)
    with torch.cuda.device(1):
        borrower = cuda_stack(32, 8, 32, 4096, capacity_chunks=512)
        assert borrower.dev.cuda_ordinal == 1
        tpc = borrower.cfg.tokens_per_chunk
        rm, stats = import_prefix(borrower.sched, "turn", tokens, shared)
        assert stats.identity_ok and stats.shared_tokens == PREFIX
        borrower.dev.wait()
        bva = borrower.dev.va(rm.vt.space.rng)
        own = chunk_view(bva, (PREFIX + NEW) // tpc, borrower.geo)[PREFIX // tpc:]
        own.copy_(torch.randn(own.shape, device="cuda:1").to(torch.bfloat16))
        q = torch.randn(1, NEW, 32, 128, device="cuda:1").to(torch.bfloat16)
        maps = kv_tensor_maps([bva], [PREFIX + NEW], borrower.geo, device="cuda:1")
        out = prefill_attention(q, maps, torch.tensor([PREFIX], dtype=torch.int32, device="cuda:1"),
                                11, borrower.geo)
        torch.cuda.synchronize()
        k_b, v_b = read_kv(bva, PREFIX + NEW, 11, borrower.geo)
    with torch.cuda.device(0):
        k_d, v_d = read_kv(dva, PREFIX, 11, donor.geo)
    assert torch.equal(k_d.cpu(), k_b[:, :PREFIX].cpu()) and torch.equal(v_d.cpu(), v_b[:, :PREFIX].cpu())
    ref = prefill_attention_ref(q[0].cpu(), k_b.cpu(), v_b.cpu(), PREFIX)
    assert rel_err(out[0].cpu(), ref) <= 2e-2
    with torch.cuda.device(1):
        borrower.sched.mark_prefilled("turn")
        borrower.sched.release("turn")
        borrower.dev.wait()
