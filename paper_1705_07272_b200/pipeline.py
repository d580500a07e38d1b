"""Host-buffer serving pipeline for the hot path: one call per step takes the frames' light
pyramids and shifts in pinned HOST memory and returns radiance in pinned HOST memory.

Plumbing only (torch streams, events and async copies); both compute steps are the C-ABI kernels
(``haar_shift_coeffs``, ``relight_vertices``).  Overlap, per step i:

    h2d stream   : light_i  -> device buffer (i % 2)            (waits until step i-2's shift read it)
    compute      : shift(light_i) ; relight chunk 0 ; relight chunk 1 ; ...
    d2h stream   :                  R chunk 0 -> host ; R chunk 1 -> host ; ...

so the H2D of step i+1 runs under step i's relight, and every radiance chunk is copied back while
the next chunk computes; H2D and D2H use different copy engines (full duplex).  Every step still
moves its own inputs in and its own result out.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import api
from .dist import allgather_band, chunk_bounds, shard_rows


class ShiftRelightPipeline:
    def __init__(self, transfer: torch.Tensor, faces: int, log2n: int, batch: int, band_levels: int,
                 chunks: int = 8, full_pyramids: bool = True):
        dev = transfer.device
        N = 1 << log2n
        self.T = transfer
        self.faces, self.log2n, self.batch = faces, log2n, batch
        self.band = band_levels
        self.k_face = 4 ** band_levels
        self.full = full_pyramids
        self.V = transfer.shape[0]
        self.light = [torch.empty((batch, faces, N * N), dtype=torch.float32, device=dev) for _ in range(2)]
        self.shifted = torch.empty((batch, faces, N * N if full_pyramids else self.k_face), dtype=torch.float32,
                                   device=dev)
        self.R = torch.empty((self.V, batch), dtype=torch.float32, device=dev)
        ws = api.haar_shift_workspace_bytes(2, log2n, faces, batch)
        self.ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
        rws = api.relight_workspace_bytes(faces, self.k_face, batch)
        self.rws = None
        if rws:
            raw = torch.empty(rws + 1024, dtype=torch.uint8, device=dev)
            self.rws = raw[(-raw.data_ptr()) % 1024:]
        self.chunks = chunk_bounds(self.V, chunks)
        self.compute = torch.cuda.current_stream(dev)
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_light_free = [torch.cuda.Event() for _ in range(2)]
        self.ev_chunk = [torch.cuda.Event() for _ in self.chunks]
        self.ev_copied = [torch.cuda.Event() for _ in self.chunks]
        self.i = 0
        self.launches = 0

    def _relight_chunk(self, s: int, n: int) -> None:
        api.relight_vertices(self.T[s:s + n], self.shifted, self.faces, self.k_face, out=self.R[s:s + n],
                             workspace=self.rws, stream=self.compute)

    def step(self, light_host: torch.Tensor, shifts, radiance_host: torch.Tensor) -> torch.cuda.Event:
        """Enqueue one step; returns an event that completes when radiance_host holds the result."""
        buf = self.i & 1
        with torch.cuda.stream(self.h2d):
            if self.i >= 2:
                self.h2d.wait_event(self.ev_light_free[buf])
            self.light[buf].copy_(light_host, non_blocking=True)
            self.ev_h2d[buf].record(self.h2d)
        self.compute.wait_event(self.ev_h2d[buf])
        api.haar_shift_coeffs(self.light[buf], shifts, 2, self.log2n if self.full else self.band, out=self.shifted,
                              workspace=self.ws, stream=self.compute)
        self.launches += api.last_launch_count()
        self.ev_light_free[buf].record(self.compute)
        for c, (s, n) in enumerate(self.chunks):
            if self.i >= 1:
                self.compute.wait_event(self.ev_copied[c])  # previous step's D2H of this chunk is done
            self._relight_chunk(s, n)
            self.launches += api.last_launch_count()
            self.ev_chunk[c].record(self.compute)
            self.d2h.wait_event(self.ev_chunk[c])
            with torch.cuda.stream(self.d2h):
                radiance_host[s:s + n].copy_(self.R[s:s + n], non_blocking=True)
                self.ev_copied[c].record(self.d2h)
        self.i += 1
        return self.ev_copied[-1]


class ShardedShiftRelightPipeline:
    """The host-buffer step at N > 1 ranks: per step, every rank copies only its own
    frames' light pyramids host -> device, shifts them to the band (``haar_shift_coeffs``), the band
    is all-gathered over NCCL / NVLink (``dist.allgather_band``, the one exchange step), and the
    rank relights its own vertex rows chunk by chunk, each chunk's radiance copied device -> host
    straight into the rank's rows of ``radiance_host`` -- a ``dist.SharedHostBuffer`` every rank
    maps -- while the next chunk computes.  The host gather therefore runs over all N PCIe links
    at once instead of funnelling the whole radiance through rank 0's.  Plumbing only; the compute
    is the C-ABI kernels.  Single rank: the same schedule with a local band copy."""

    def __init__(self, transfer_local: torch.Tensor, faces: int, log2n: int, batch: int, band_levels: int,
                 total_rows: int, chunks: int = 4, group=None):
        import torch.distributed as dist
        dev = transfer_local.device
        N = 1 << log2n
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.row0, count = shard_rows(total_rows, world, rank)
        if transfer_local.shape[0] != count:
            raise ValueError(f"rank {rank}: expected {count} transfer rows, got {transfer_local.shape[0]}")
        self.f0, self.fn = shard_rows(batch, world, rank)
        self.T = transfer_local
        self.faces, self.log2n, self.batch, self.band = faces, log2n, batch, band_levels
        self.k_face = 4 ** band_levels
        self.light = [torch.empty((max(self.fn, 1), faces, N * N), dtype=torch.float32, device=dev) for _ in range(2)]
        self.band_local = torch.empty((max(self.fn, 1), faces, self.k_face), dtype=torch.float32, device=dev)
        self.band_full = torch.empty((batch, faces, self.k_face), dtype=torch.float32, device=dev)
        self.R = torch.empty((count, batch), dtype=torch.float32, device=dev)
        self.ws = torch.empty(max(api.haar_shift_workspace_bytes(2, log2n, faces, max(self.fn, 1)), 1),
                              dtype=torch.uint8, device=dev)
        rws = api.relight_workspace_bytes(faces, self.k_face, batch)
        self.rws = None
        if rws:
            raw = torch.empty(rws + 1024, dtype=torch.uint8, device=dev)
            self.rws = raw[(-raw.data_ptr()) % 1024:]
        self.chunks = chunk_bounds(count, chunks)
        self.compute = torch.cuda.current_stream(dev)
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_light_free = [torch.cuda.Event() for _ in range(2)]
        self.ev_chunk = [torch.cuda.Event() for _ in self.chunks]
        self.ev_copied = [torch.cuda.Event() for _ in self.chunks]
        self.ev_done = torch.cuda.Event()
        self.i = 0
        self.launches = 0

    def h2d_bytes(self) -> int:
        return self.fn * self.faces * (1 << (2 * self.log2n)) * 4

    def d2h_bytes(self) -> int:
        return self.R.numel() * 4

    def step(self, light_host: torch.Tensor, shifts, radiance_host: torch.Tensor) -> torch.cuda.Event:
        """light_host: pinned [batch][faces][N*N] (this rank copies its frames); shifts: host
        [batch][faces][2]; radiance_host: the shared pinned [total_rows][batch] buffer.  Returns an
        event that completes when this rank's rows are in radiance_host."""
        buf = self.i & 1
        f0, fn = self.f0, self.fn
        if fn:
            with torch.cuda.stream(self.h2d):
                if self.i >= 2:
                    self.h2d.wait_event(self.ev_light_free[buf])
                self.light[buf][:fn].copy_(light_host[f0:f0 + fn], non_blocking=True)
                self.ev_h2d[buf].record(self.h2d)
            self.compute.wait_event(self.ev_h2d[buf])
            sh = np.asarray(shifts, dtype=np.float64)[f0:f0 + fn]
            api.haar_shift_coeffs(self.light[buf][:fn], sh, 2, self.band, out=self.band_local[:fn],
                                  workspace=self.ws, stream=self.compute)
            self.launches += api.last_launch_count()
        self.ev_light_free[buf].record(self.compute)
        with torch.cuda.stream(self.compute):
            allgather_band(self.band_local[:fn], self.band_full, group=self.group)
        for c, (s, n) in enumerate(self.chunks):
            if self.i >= 1:
                self.compute.wait_event(self.ev_copied[c])   # the previous step's D2H of this chunk is done
            api.relight_vertices(self.T[s:s + n], self.band_full, self.faces, self.k_face, out=self.R[s:s + n],
                                 workspace=self.rws, stream=self.compute)
            self.launches += api.last_launch_count()
            self.ev_chunk[c].record(self.compute)
            self.d2h.wait_event(self.ev_chunk[c])
            with torch.cuda.stream(self.d2h):
                g = self.row0 + s
                radiance_host[g:g + n].copy_(self.R[s:s + n], non_blocking=True)
                self.ev_copied[c].record(self.d2h)
        self.ev_done.record(self.d2h)
        self.i += 1
        return self.ev_done


class ShiftTripleRelightPipeline(ShiftRelightPipeline):
    """The same host pipeline with the triple-product relight (row f3): per-vertex BRDF and
    visibility in the qtree layout (``relight_vertices_triple``) instead of one transfer matrix."""

    def __init__(self, brdf_q: torch.Tensor, vis_q: torch.Tensor, faces: int, log2n: int, batch: int,
                 band_levels: int, chunks: int = 8, full_pyramids: bool = False):
        super().__init__(brdf_q, faces, log2n, batch, band_levels, chunks, full_pyramids)
        self.vis = vis_q
        rows = max(n for _, n in self.chunks)
        need = api.relight_triple_workspace_bytes(rows, faces, self.k_face, batch)
        raw = torch.empty(need + 1024, dtype=torch.uint8, device=brdf_q.device)
        self.tws = raw[(-raw.data_ptr()) % 1024:]

    def _relight_chunk(self, s: int, n: int) -> None:
        api.relight_vertices_triple(self.T[s:s + n], self.vis[s:s + n], self.shifted, self.faces, self.k_face,
                                    out=self.R[s:s + n], workspace=self.tws, stream=self.compute)


class ShiftSparseRelightPipeline(ShiftRelightPipeline):
    """The same host pipeline with the sparse-transfer relight (row f2): per-vertex (index, value)
    pairs over the full shifted pyramids (``relight_vertices_sparse``).  Each chunk's call
    re-transposes the light (a ~0.03 ms pass at c5s), so fewer, larger chunks are used."""

    def __init__(self, indices: torch.Tensor, values: torch.Tensor, faces: int, log2n: int, batch: int,
                 chunks: int = 4):
        super().__init__(values, faces, log2n, batch, log2n, chunks, full_pyramids=True)
        self.rws = None   # the dense relight's workspace is not used here
        self.idx = indices
        need = api.relight_sparse_workspace_bytes(faces * (1 << (2 * log2n)), batch)
        self.sws = torch.empty(need, dtype=torch.uint8, device=values.device)

    def _relight_chunk(self, s: int, n: int) -> None:
        api.relight_vertices_sparse(self.idx[s:s + n], self.T[s:s + n], self.shifted, out=self.R[s:s + n],
                                    workspace=self.sws, stream=self.compute)


class RotatePipeline:
    """Host-buffer rotation of lat-long maps (row f1): the maps are processed in chunks, chunk k+1's
    H2D and chunk k-1's D2H (two copy streams, two copy engines) running under chunk k's
    ``haar_rotate_coeffs``.  Plumbing only."""

    def __init__(self, maps: int, log2n: int, device, chunks: int = 4):
        self.N2 = 1 << (2 * log2n)
        self.log2n = log2n
        self.chunks = chunk_bounds(maps, chunks)
        self.x = torch.empty((maps, self.N2), dtype=torch.float32, device=device)
        self.y = torch.empty_like(self.x)
        rows = max(n for _, n in self.chunks)
        self.ws = torch.empty(api.haar_rotate_workspace_bytes(log2n, rows), dtype=torch.uint8, device=device)
        self.compute = torch.cuda.current_stream(device)
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.ev_in = [torch.cuda.Event() for _ in self.chunks]
        self.ev_done = [torch.cuda.Event() for _ in self.chunks]
        self.ev_out = [torch.cuda.Event() for _ in self.chunks]
        self.i = 0

    def step(self, maps_host: torch.Tensor, angles, out_host: torch.Tensor) -> torch.cuda.Event:
        """Enqueue one call; returns an event that completes when out_host holds the result."""
        ang = np.asarray(angles, dtype=np.float64).reshape(-1, 2)
        for c, (s, n) in enumerate(self.chunks):
            with torch.cuda.stream(self.h2d):
                if self.i >= 1:
                    self.h2d.wait_event(self.ev_done[c])   # the previous call's rotation read x[s:s+n]
                self.x[s:s + n].copy_(maps_host[s:s + n], non_blocking=True)
                self.ev_in[c].record(self.h2d)
        for c, (s, n) in enumerate(self.chunks):
            self.compute.wait_event(self.ev_in[c])
            if self.i >= 1:
                self.compute.wait_event(self.ev_out[c])    # the previous call's D2H of y[s:s+n] is done
            api.haar_rotate_coeffs(self.x[s:s + n], ang[s:s + n], out=self.y[s:s + n], workspace=self.ws,
                                   stream=self.compute)
            self.ev_done[c].record(self.compute)
            self.d2h.wait_event(self.ev_done[c])
            with torch.cuda.stream(self.d2h):
                out_host[s:s + n].copy_(self.y[s:s + n], non_blocking=True)
                self.ev_out[c].record(self.d2h)
        self.i += 1
        return self.ev_out[-1]
