"""Multi-GPU data parallelism over vertex rows.

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing:

* vertex rows are contiguous blocks [start_r, start_r + count_r) per rank (``shard_rows``); the
  transfer rows T are generated in place on their rank from the counter hash keyed by the GLOBAL
  row id, so every shard is bitwise the 1-GPU matrix's slice and never moves;
* the shifted lighting band is computed sharded by frame (each rank shifts its ``frame_shard`` of the
  batch) and all-gathered (``allgather_band``, NCCL over NVLink) -- the one exchange step into the
  relight; ``broadcast_band`` (rank 0 shifts everything) is kept for single-frame batches;
* radiance reaches rank 0 in one of two ways:
  - fused (``open_peer_view`` + ``relight_into_peer``, the default of bench.py): rank 0's radiance
    buffer is opened in every rank through CUDA IPC and each rank's relight kernel stores its
    rows straight into it over NVLink / NVSwitch from the epilogue -- the gather IS the relight's
    output write, no separate collective, no staging copy; ``rows_landed_fence`` (a one-element
    all-reduce on the stream) orders rank 0's later work after every rank's rows, stream-ordered;
  - host buffers (``SharedHostBuffer`` + pipeline.ShardedShiftRelightPipeline): every rank copies
    its own rows device->host into one shared page-locked host array, chunk by chunk under its
    relight, so all N PCIe links carry the gather;
  - NCCL (``relight_and_gather``, the baseline and the fallback): chunk i is gathered on the NCCL
    stream while chunk i+1 is relit, so the gather overlaps the HBM-bound relight.

Per-row results do not depend on the sharding (each row's reduction order is fixed inside the
kernels), so the gathered R equals the 1-GPU R bit for bit.

The compute step is injected (``relight_fn``) so the communication logic is testable on CPU with
gloo; on the GPU it is always the C-ABI ``relight_vertices``.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


def shard_rows(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-equal blocks: the first (total % world) ranks get one extra row."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start, count


def max_shard(total: int, world: int) -> int:
    return -(-total // world)


def chunk_bounds(count: int, chunks: int) -> List[Tuple[int, int]]:
    """Split [0, count) into ``chunks`` contiguous near-equal pieces (empty pieces dropped)."""
    chunks = max(1, min(chunks, max(count, 1)))
    out = []
    for c in range(chunks):
        s, n = shard_rows(count, chunks, c)
        if n > 0:
            out.append((s, n))
    return out


def broadcast_band(band: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Broadcast the shifted lighting band (rank ``src`` computed it) to every rank in place."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(band, src=src, group=group)
    return band


def frame_shard(batch: int, group=None) -> Tuple[int, int]:
    """This rank's contiguous block of light frames for the sharded shift ([start, start+count))."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return shard_rows(batch, world, rank)


def allgather_band(band_local: torch.Tensor, band_full: torch.Tensor, group=None) -> torch.Tensor:
    """The shift sharded by frame: every rank shifted its ``frame_shard`` frames into ``band_local``
    ([count][faces][stride]); gather all of them into ``band_full`` ([batch][faces][stride]) on every
    rank.  Equal shards go through one all_gather_into_tensor (NCCL over NVLink); uneven ones are
    padded to the largest shard."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    B = band_full.shape[0]
    if world == 1:
        band_full.copy_(band_local)
        return band_full
    ms = max_shard(B, world)
    if B % world == 0:
        dist.all_gather_into_tensor(band_full, band_local.contiguous(), group=group)
        return band_full
    pad = torch.zeros((ms,) + tuple(band_local.shape[1:]), dtype=band_local.dtype, device=band_local.device)
    pad[: band_local.shape[0]].copy_(band_local)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    for r in range(world):
        s, c = shard_rows(B, world, r)
        band_full[s:s + c].copy_(parts[r][:c])
    return band_full


def relight_and_gather(transfer_local: torch.Tensor, band: torch.Tensor, total_rows: int,
                       relight_fn: Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None],
                       radiance_full: Optional[torch.Tensor] = None, chunks: int = 4,
                       gather: bool = True, group=None) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """Relight this rank's rows chunk by chunk and gather radiance into rank 0, overlapping the
    gather of chunk i with the relight of chunk i+1.

    transfer_local: [count_r][K] this rank's rows; band: [B][F][stride] (already broadcast);
    relight_fn(T_chunk, band, R_chunk_out) fills R_chunk_out [rows][B].
    radiance_full (rank 0, [total_rows][B]) receives every rank's rows at their global offsets.
    Returns (local radiance [count_r][B], radiance_full or None).
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = band.shape[0]
    start, count = shard_rows(total_rows, world, rank)
    if transfer_local.shape[0] != count:
        raise ValueError(f"rank {rank}: expected {count} transfer rows, got {transfer_local.shape[0]}")
    local = torch.empty((count, B), dtype=torch.float32, device=transfer_local.device)
    if world == 1 or not gather:
        for s, n in chunk_bounds(count, chunks):
            relight_fn(transfer_local[s:s + n], band, local[s:s + n])
        if world == 1 and radiance_full is not None:
            radiance_full.copy_(local)
        return local, radiance_full
    # every rank runs the same chunk schedule: chunk c of every rank has the same size when shards
    # are padded to max_shard -> one all_gather per chunk (NCCL collectives need equal sizes)
    ms = max_shard(total_rows, world)
    sched = chunk_bounds(ms, chunks)
    recv = None
    if rank == 0:
        if radiance_full is None:
            radiance_full = torch.empty((total_rows, B), dtype=torch.float32, device=transfer_local.device)
    pending = []
    for s, n in sched:
        lo, hi = min(s, count), min(s + n, count)
        if hi > lo:
            relight_fn(transfer_local[lo:hi], band, local[lo:hi])
        send = torch.zeros((n, B), dtype=torch.float32, device=local.device)
        if hi > lo:
            send[: hi - lo].copy_(local[lo:hi])
        recv = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
        work = dist.gather(send, gather_list=recv, dst=0, group=group, async_op=True)
        pending.append((work, s, n, recv, send))
    for work, s, n, recv_l, _send in pending:
        work.wait()
        if rank == 0:
            for r in range(world):
                rs, rc = shard_rows(total_rows, world, r)
                lo, hi = min(s, rc), min(s + n, rc)
                if hi > lo:
                    radiance_full[rs + lo:rs + hi].copy_(recv_l[r][: hi - lo])
    return local, radiance_full


def open_peer_view(radiance_full: Optional[torch.Tensor], shape, device: torch.device, group=None) -> torch.Tensor:
    """Every rank gets a tensor aliasing rank 0's ``radiance_full`` (CUDA IPC through torch's own
    storage sharing; peer access to rank 0's device is enabled first).  Rank 0 passes its buffer,
    the others pass None.  Raises if the devices cannot reach each other (callers fall back to
    ``relight_and_gather``)."""
    from torch.multiprocessing.reductions import reduce_tensor

    from . import api
    rank = dist.get_rank(group)
    obj = [None]
    if rank == 0:
        fn, args = reduce_tensor(radiance_full)
        obj = [(fn, args, radiance_full.device.index)]
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank == 0:
        return radiance_full
    fn, args, dev0 = obj[0]
    api.enable_peer_access(dev0)
    view = fn(*args)
    if tuple(view.shape) != tuple(shape):
        raise RuntimeError("peer view has the wrong shape")
    return view


def rows_landed_fence(flag: torch.Tensor, group=None) -> None:
    """Stream-ordered completion of the fused relight + gather: a one-element all-reduce enqueued
    on every rank's current stream after its relight.  It completes on rank 0 only once every
    rank's relight kernel (whose epilogue stored into rank 0's buffer) has finished, so work that
    rank 0 enqueues after it sees every row -- no host synchronisation, no host barrier.
    ``flag``: a persistent one-element device tensor (int32)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flag, group=group)


class SharedHostBuffer:
    """A float32 array in POSIX shared memory (/dev/shm) mapped by every rank of the node and
    page-locked in each (cudaHostRegister), so that every rank's device->host copies land in one
    host array over its own PCIe link: the N>1 radiance gather on the host side.  Rank 0 creates
    the file, the others map it after a broadcast of its name; ``close`` unmaps and unpins (rank 0
    unlinks)."""

    def __init__(self, shape, group=None, pin: bool = True):
        import mmap
        import os
        import numpy as np
        self.shape = tuple(int(x) for x in shape)
        self.nbytes = int(np.prod(self.shape)) * 4
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        name = [None]
        if self.rank == 0:
            name = [f"/dev/shm/hs_radiance_{os.getpid()}_{id(self)}"]
            with open(name[0], "wb") as fh:
                fh.truncate(self.nbytes)
        if dist.is_initialized():
            dist.broadcast_object_list(name, src=0, group=group)
        self.path = name[0]
        self._fh = open(self.path, "r+b")
        self._mm = mmap.mmap(self._fh.fileno(), self.nbytes)
        self.array = np.ndarray(self.shape, dtype=np.float32, buffer=self._mm)
        self.tensor = torch.from_numpy(self.array)
        self.pinned = False
        if pin and torch.cuda.is_available():
            err = torch.cuda.cudart().cudaHostRegister(self.tensor.data_ptr(), self.nbytes, 0)
            if int(err) != 0:
                raise RuntimeError(f"cudaHostRegister of the shared radiance buffer failed ({err})")
            self.pinned = True

    def close(self) -> None:
        import os
        if self.pinned:
            torch.cuda.cudart().cudaHostUnregister(self.tensor.data_ptr())
            self.pinned = False
        self.tensor = None
        self.array = None
        self._mm.close()
        self._fh.close()
        if dist.is_initialized():
            dist.barrier(group=self.group)
        if self.rank == 0 and os.path.exists(self.path):
            os.unlink(self.path)


def relight_into_peer(transfer_local: torch.Tensor, band: torch.Tensor, total_rows: int,
                      relight_fn: Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None],
                      radiance_view: torch.Tensor, group=None) -> None:
    """The fused relight + gather: this rank's rows are written by the relight kernel directly at
    their global offset of rank 0's radiance (``radiance_view`` from ``open_peer_view``).  The
    caller orders completion (``rows_landed_fence``) before rank 0 reads the buffer."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    start, count = shard_rows(total_rows, world, rank)
    if transfer_local.shape[0] != count:
        raise ValueError(f"rank {rank}: expected {count} transfer rows, got {transfer_local.shape[0]}")
    if count:
        relight_fn(transfer_local, band, radiance_view[start:start + count])
