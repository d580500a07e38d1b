"""Multi-GPU plumbing on CPU (-m "not gpu"): world-size-2 (and 3) gloo process groups exercise the
vertex-row sharding, the band broadcast and the chunked, overlapped radiance gather of
paper_1705_07272_b200.dist.  The per-rank compute is an injected CPU double (a float64 matmul), not
the oracle and not the product kernel; what is under test is that every rank's rows land at
their global offsets in rank 0's radiance and that the result equals the unsharded one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_07272_b200 import dist as hsdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relight_double(T, band, R):
    B = band.shape[0]
    K = T.shape[1]
    R.copy_((T.double() @ band.reshape(B, -1)[:, :K].double().T).float())


def _worker(rank, world, port, V, F, kf, B, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        T_full = torch.randn(V, F * kf, generator=g)
        band_full = torch.randn(B, F, kf, generator=g)
        start, count = hsdist.shard_rows(V, world, rank)
        T_local = T_full[start:start + count].contiguous()
        band = band_full.clone() if rank == 0 else torch.zeros(B, F, kf)
        hsdist.broadcast_band(band)
        assert torch.equal(band, band_full)
        R_full = torch.full((V, B), float("nan")) if rank == 0 else None
        local, full = hsdist.relight_and_gather(T_local, band, V, _relight_double, R_full, chunks=chunks)
        ref_local = torch.empty(count, B)
        _relight_double(T_local, band_full, ref_local)
        assert torch.equal(local, ref_local)
        if rank == 0:
            ref = torch.empty(V, B)
            _relight_double(T_full, band_full, ref)
            q.put(("ok", bool(torch.equal(full, ref)), float((full - ref).abs().max())))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,V,chunks", [(2, 1001, 4), (2, 64, 1), (3, 1000, 3), (2, 5, 4)])
def test_sharded_relight_gather_equals_unsharded(world, V, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, 6, 16, 8, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    oks = [m for m in msgs if m[0] == "ok"]
    assert oks and oks[0][1], msgs


def test_shard_rows_partition():
    for V in [0, 1, 7, 1000, 1_000_000]:
        for world in [1, 2, 3, 8]:
            pieces = [hsdist.shard_rows(V, world, r) for r in range(world)]
            assert sum(c for _, c in pieces) == V
            pos = 0
            for s, c in pieces:
                assert s == pos
                pos += c
            assert max(c for _, c in pieces) - min(c for _, c in pieces) <= 1
            assert hsdist.max_shard(V, world) == max(c for _, c in pieces)


def test_chunk_bounds():
    assert hsdist.chunk_bounds(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert hsdist.chunk_bounds(2, 4) == [(0, 1), (1, 1)]
    assert hsdist.chunk_bounds(0, 4) == []
    with pytest.raises(ValueError):
        hsdist.shard_rows(10, 2, 2)


def _band_worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(3)
        full = torch.randn(B, 6, 16, generator=g)
        s, c = hsdist.frame_shard(B)
        assert (s, c) == hsdist.shard_rows(B, world, rank)
        got = torch.full_like(full, float("nan"))
        hsdist.allgather_band(full[s:s + c].clone(), got)
        q.put(("ok", rank, bool(torch.equal(got, full))))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, 64), (3, 64), (2, 5)])
def test_sharded_shift_band_allgather(world, B):
    """every rank shifts its frames; the all-gathered band equals the unsharded one on every rank
    (equal shards: one all_gather_into_tensor; uneven: padded all_gather)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert len([m for m in msgs if m[0] == "ok" and m[2]]) == world, msgs


def _shared_worker(rank, world, port, V, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf = hsdist.SharedHostBuffer((V, B), pin=False)
        s, c = hsdist.shard_rows(V, world, rank)
        buf.tensor[s:s + c] = torch.arange(s * B, (s + c) * B, dtype=torch.float32).reshape(c, B)  # this rank's rows
        flag = torch.zeros(1, dtype=torch.int32)
        hsdist.rows_landed_fence(flag)          # gloo: a blocking all-reduce
        dist.barrier()
        if rank == 0:
            want = torch.arange(V * B, dtype=torch.float32).reshape(V, B)
            q.put(("ok", bool(torch.equal(buf.tensor, want))))
        path = buf.path
        buf.close()
        if rank == 0:
            q.put(("unlinked", not os.path.exists(path)))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,V,B", [(2, 1001, 4), (3, 10, 64)])
def test_shared_host_buffer_gathers_every_rank(world, V, B):
    """the N>1 host gather: each rank writes its own rows into one /dev/shm array mapped by all
    ranks; rank 0 sees every row; the file is removed on close"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, V, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert ("ok", True) in msgs and ("unlinked", True) in msgs, msgs
