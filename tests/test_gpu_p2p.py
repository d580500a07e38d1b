"""The fused relight + gather path of SURVEY §8(e) (-m gpu): rank 0's radiance buffer is opened in
the other ranks through CUDA IPC (paper_1705_07272_b200.dist.open_peer_view) and each rank's
relight_vertices kernel stores its rows straight into it.  The pool has one GPU, so the two ranks
share cuda:0 here (gloo for the handle exchange and the barrier; no kernel waits on another rank's
kernel); on a multi-GPU node the same code path writes over NVLink after hs_enable_peer_access.
Checked: every row lands at its global offset and equals the fp64 oracle (rel-L2 <= 1e-5)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, V, B, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import synth
    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200 import dist as hsdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        F, kf = 6, 256
        start, count = hsdist.shard_rows(V, world, rank)
        T = torch.empty((count, F * kf), dtype=torch.float32, device=dev)
        hs.hs_fill_transfer(T, start, F, kf, synth.SEED_BASE + 9, synth.STREAM_T)
        band = torch.from_numpy(synth.light_pyramids(31, B, F, 4)).to(dev)
        R_full = torch.full((V, B), float("nan"), device=dev) if rank == 0 else None
        view = hsdist.open_peer_view(R_full, (V, B), dev)

        def relight_fn(Tc, bnd, Rc):
            hs.relight_vertices(Tc, bnd, F, kf, out=Rc)

        hsdist.relight_into_peer(T, band, V, relight_fn, view)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            from oracle import relight as orelight
            ref = orelight.relight(synth.transfer_rows(synth.SEED_BASE + 9, 0, V, F, kf),
                                   synth.light_pyramids(31, B, F, 4), F, kf)
            got = R_full.cpu().numpy()
            ok = bool(np.isfinite(got).all()) and float(np.linalg.norm(got - ref) / np.linalg.norm(ref)) <= 1e-5
            q.put(("ok", ok))
        dist.barrier()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), rank))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,V,B", [(2, 1001, 4), (3, 640, 64)])
def test_relight_writes_into_rank0_buffer(world, V, B):
    """B * 4 bytes per row keeps every shard's first row 16-byte aligned (the ABI requires it)"""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    assert any(m[0] == "ok" and m[1] for m in msgs), msgs
