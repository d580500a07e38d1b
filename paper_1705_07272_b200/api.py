"""Python binding of the C ABI (include/haarshift.h): marshalling of torch tensors to pointers,
nothing else.  All tensors passed as device arguments must be CUDA float32, contiguous and 16-byte
aligned; results are new tensors unless ``out=`` is given.  Work is enqueued on the current torch
CUDA stream (or ``stream=``)."""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from ._lib import check, load


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _log2n_pow4(K: int, what: str) -> int:
    """log2 N of a face of K = 4**log2n coefficients; ValueError otherwise."""
    n = int(K).bit_length() - 1
    if K < 4 or n % 2 or (1 << n) != K:
        raise ValueError(f"{what} must hold 4**log2n coefficients (got {K})")
    return n // 2


def _out(out: Optional[torch.Tensor], shape, device, name: str = "out") -> torch.Tensor:
    """a new float32 result tensor, or the caller's `out` checked like every other device argument"""
    if out is None:
        return torch.empty(tuple(shape), dtype=torch.float32, device=device)
    _dev_f32(out, name)
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(out.shape)}")
    return out


def enable_peer_access(peer_device: int) -> None:
    """Allow kernels on the current device to access `peer_device`'s memory (include/haarshift.h)."""
    check("hs_enable_peer_access", load().hs_enable_peer_access(int(peer_device)))


def last_launch_count() -> int:
    """Kernel launches enqueued by the most recent C-ABI call on this thread."""
    return int(load().hs_last_launch_count())


def haar_shift_workspace_bytes(ndim: int, log2n: int, faces: int, batch: int) -> int:
    return int(load().haar_shift_workspace_bytes(ndim, log2n, faces, batch))


def relight_shifted_workspace_bytes(num_vertices: int, faces: int, log2n: int) -> int:
    return int(load().relight_shifted_workspace_bytes(num_vertices, faces, log2n))


def haar_shift_coeffs(coeffs: torch.Tensor, shifts, ndim: int = 2, band_levels: Optional[int] = None,
                      out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """coeffs [batch][faces][K] (K = N*N in 2D, N in 1D) -> shifted pyramids [batch][faces][Kb].

    shifts: host array-like [batch][faces][ndim] (fp64; (sy, sx) in 2D)."""
    lib = load()
    _dev_f32(coeffs, "coeffs")
    if coeffs.dim() != 3:
        raise ValueError("coeffs must be [batch][faces][K]")
    B, F, K = coeffs.shape
    if ndim == 2:
        log2n = _log2n_pow4(K, "2D faces")
    else:
        log2n = int(K).bit_length() - 1
        if (1 << log2n) != K:
            raise ValueError("1D signals must hold 2**log2n coefficients")
    band = log2n if band_levels is None else int(band_levels)
    kb = (4 if ndim == 2 else 2) ** band
    sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.float64).reshape(B, F, ndim))
    out = _out(out, (B, F, kb), coeffs.device)
    need = haar_shift_workspace_bytes(ndim, log2n, F, B)
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.empty(need, dtype=torch.uint8, device=coeffs.device)
    ws_ptr = workspace.data_ptr() if (need and workspace is not None) else None
    st = lib.haar_shift_coeffs(coeffs.data_ptr(), out.data_ptr(), ndim, log2n, F, B,
                               sh.ctypes.data_as(ctypes.c_void_p), band, ws_ptr, need, _stream_ptr(stream))
    check("haar_shift_coeffs", st)
    return out


def haar_shift_coarse_workspace_bytes(in_log2n: int, start_level: int, faces: int, batch: int) -> int:
    return int(load().haar_shift_coarse_workspace_bytes(in_log2n, start_level, faces, batch))


def haar_shift_coeffs_coarse(coeffs: torch.Tensor, shifts, start_level: int, band_levels: Optional[int] = None,
                             out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Coarse-start shift: coeffs [batch][faces][4**n] -> the shifted level-L approximation,
    [batch][faces][4**band] (band <= L, default L).  shifts: host [batch][faces][2] in pixels."""
    lib = load()
    _dev_f32(coeffs, "coeffs")
    if coeffs.dim() != 3:
        raise ValueError("coeffs must be [batch][faces][K]")
    B, F, K = coeffs.shape
    n = _log2n_pow4(K, "2D faces")
    band = start_level if band_levels is None else int(band_levels)
    sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.float64).reshape(B, F, 2))
    out = _out(out, (B, F, 4 ** band), coeffs.device)
    need = haar_shift_coarse_workspace_bytes(n, start_level, F, B)
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.empty(need, dtype=torch.uint8, device=coeffs.device)
    st = lib.haar_shift_coeffs_coarse(coeffs.data_ptr(), out.data_ptr(), n, start_level, F, B,
                                      sh.ctypes.data_as(ctypes.c_void_p), band,
                                      workspace.data_ptr() if need else None, need, _stream_ptr(stream))
    check("haar_shift_coeffs_coarse", st)
    return out


def haar_rotate_workspace_bytes(log2n: int, batch: int) -> int:
    return int(load().haar_rotate_workspace_bytes(log2n, batch))


def haar_rotate_coeffs(coeffs: torch.Tensor, angles, out: Optional[torch.Tensor] = None,
                       workspace: Optional[torch.Tensor] = None,
                       stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """coeffs [batch][N*N] (HAAR1 lat-long maps) -> rotated pyramids [batch][N*N]; angles host
    [batch][2] (alpha elevation about X, beta azimuth) in radians (include/haarshift.h)."""
    lib = load()
    _dev_f32(coeffs, "coeffs")
    B = coeffs.shape[0]
    K = coeffs.numel() // B
    n = _log2n_pow4(K, "maps")
    ang = np.ascontiguousarray(np.asarray(angles, dtype=np.float64).reshape(B, 2))
    out = _out(out, coeffs.shape, coeffs.device)
    need = haar_rotate_workspace_bytes(n, B)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=coeffs.device)
    st = lib.haar_rotate_coeffs(coeffs.data_ptr(), out.data_ptr(), n, B, ang.ctypes.data_as(ctypes.c_void_p),
                                workspace.data_ptr(), need, _stream_ptr(stream))
    check("haar_rotate_coeffs", st)
    return out


def relight_workspace_bytes(faces: int, k_face: int, batch: int) -> int:
    return int(load().relight_workspace_bytes(faces, k_face, batch))


def relight_vertices(transfer: torch.Tensor, light: torch.Tensor, faces: int, k_face: int,
                     out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """transfer [V][faces*k_face], light [batch][faces][stride >= k_face] -> radiance [V][batch]."""
    lib = load()
    _dev_f32(transfer, "transfer")
    _dev_f32(light, "light")
    V = transfer.shape[0]
    if transfer.numel() != V * faces * k_face:
        raise ValueError("transfer must be [V][faces*k_face]")
    if light.dim() != 3 or light.shape[1] != faces:
        raise ValueError("light must be [batch][faces][stride]")
    B, _, stride = light.shape
    out = _out(out, (V, B), transfer.device)
    need = relight_workspace_bytes(faces, k_face, B)
    ws_ptr = None
    if need:
        if workspace is None or workspace.numel() * workspace.element_size() < need or workspace.data_ptr() % 1024:
            workspace = torch.empty(need, dtype=torch.uint8, device=transfer.device)   # allocator: 512B+ aligned
            if workspace.data_ptr() % 1024:
                workspace = torch.empty(need + 1024, dtype=torch.uint8, device=transfer.device)
                workspace = workspace[(-workspace.data_ptr()) % 1024:]
        ws_ptr = workspace.data_ptr()
    st = lib.relight_vertices(transfer.data_ptr(), V, faces, k_face, light.data_ptr(), stride, B, out.data_ptr(),
                              ws_ptr, need, _stream_ptr(stream))
    check("relight_vertices", st)
    return out


def relight_vertices_shifted(transfer: torch.Tensor, light: torch.Tensor, vertex_shifts: torch.Tensor,
                             out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """transfer [V][faces*N*N], light [faces][N*N], vertex_shifts [V][2] (device fp32) -> [V]."""
    lib = load()
    _dev_f32(transfer, "transfer")
    _dev_f32(light, "light")
    _dev_f32(vertex_shifts, "vertex_shifts")
    if light.dim() != 2:
        raise ValueError("light must be [faces][N*N]")
    F, K = light.shape
    n = _log2n_pow4(K, "light faces")
    V = transfer.shape[0]
    if transfer.numel() != V * F * K or tuple(vertex_shifts.shape) != (V, 2):
        raise ValueError("transfer must be [V][faces*N*N] and vertex_shifts [V][2]")
    out = _out(out, (V,), transfer.device)
    need = relight_shifted_workspace_bytes(V, F, n)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=transfer.device)
    st = lib.relight_vertices_shifted(transfer.data_ptr(), V, F, light.data_ptr(), n, vertex_shifts.data_ptr(),
                                      out.data_ptr(), workspace.data_ptr(), need, _stream_ptr(stream))
    check("relight_vertices_shifted", st)
    return out


def relight_sparse_workspace_bytes(total_coeffs: int, batch: int) -> int:
    return int(load().relight_sparse_workspace_bytes(total_coeffs, batch))


def relight_vertices_sparse(indices: torch.Tensor, values: torch.Tensor, light: torch.Tensor,
                            out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """indices int32 / values fp32 [V][K_s], light [batch][...] (flattened to [batch][C]) -> [V][batch]."""
    lib = load()
    if indices.dtype != torch.int32 or not indices.is_cuda or not indices.is_contiguous():
        raise TypeError("indices must be a contiguous CUDA int32 tensor")
    _dev_f32(values, "values")
    _dev_f32(light, "light")
    if indices.dim() != 2 or tuple(values.shape) != tuple(indices.shape):
        raise ValueError("indices and values must both be [V][K_s]")
    V, ks = indices.shape
    B = light.shape[0]
    C = light.numel() // B
    out = _out(out, (V, B), values.device)
    need = relight_sparse_workspace_bytes(C, B)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=values.device)
    st = lib.relight_vertices_sparse(indices.data_ptr(), values.data_ptr(), V, ks, light.data_ptr(), C, B,
                                     out.data_ptr(), workspace.data_ptr(), need, _stream_ptr(stream))
    check("relight_vertices_sparse", st)
    return out


def _aligned_workspace(need: int, workspace: Optional[torch.Tensor], device) -> torch.Tensor:
    if workspace is not None and workspace.numel() * workspace.element_size() >= need and workspace.data_ptr() % 1024 == 0:
        return workspace
    ws = torch.empty(need + 1024, dtype=torch.uint8, device=device)
    return ws[(-ws.data_ptr()) % 1024:]


def haar_pack_qtree(coeffs: torch.Tensor, log2k: int, out: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """coeffs [rows][faces][stride] (HAAR1, prefix 4**log2k used) -> qtree layout [rows][faces*4**log2k]
    (include/haarshift.h haar_pack_qtree)."""
    lib = load()
    _dev_f32(coeffs, "coeffs")
    if coeffs.dim() != 3:
        raise ValueError("coeffs must be [rows][faces][stride]")
    rows, F, stride = coeffs.shape
    kf = 4 ** log2k
    out = _out(out, (rows, F * kf), coeffs.device)
    st = lib.haar_pack_qtree(coeffs.data_ptr(), rows, F, stride, log2k, out.data_ptr(), _stream_ptr(stream))
    check("haar_pack_qtree", st)
    return out


def relight_triple_workspace_bytes(num_vertices: int, faces: int, k_face: int, batch: int) -> int:
    return int(load().relight_triple_workspace_bytes(num_vertices, faces, k_face, batch))


def relight_vertices_triple(brdf_q: torch.Tensor, vis_q: torch.Tensor, light: torch.Tensor, faces: int, k_face: int,
                            out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """brdf_q, vis_q [V][faces*k_face] (qtree layout), light [batch][faces][stride >= k_face] (HAAR1)
    -> radiance [V][batch] = sum_f integral of L * rho * V (triple product, eq:tripleSum)."""
    lib = load()
    _dev_f32(brdf_q, "brdf_q")
    _dev_f32(vis_q, "vis_q")
    _dev_f32(light, "light")
    V = brdf_q.shape[0]
    if brdf_q.numel() != V * faces * k_face or vis_q.shape != brdf_q.shape:
        raise ValueError("brdf_q and vis_q must be [V][faces*k_face]")
    if light.dim() != 3 or light.shape[1] != faces:
        raise ValueError("light must be [batch][faces][stride]")
    B, _, stride = light.shape
    out = _out(out, (V, B), brdf_q.device)
    need = relight_triple_workspace_bytes(V, faces, k_face, B)
    workspace = _aligned_workspace(need, workspace, brdf_q.device)
    st = lib.relight_vertices_triple(brdf_q.data_ptr(), vis_q.data_ptr(), V, faces, k_face, light.data_ptr(), stride,
                                     B, out.data_ptr(), workspace.data_ptr(), need, _stream_ptr(stream))
    check("relight_vertices_triple", st)
    return out


def relight_brdf_rotated_workspace_bytes(log2n: int, log2k: int, batch: int) -> int:
    return int(load().relight_brdf_rotated_workspace_bytes(log2n, log2k, batch))


def relight_vertices_brdf_rotated(brdf: torch.Tensor, normals, vis_q: torch.Tensor, light: torch.Tensor, log2k: int,
                                  out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """brdf [N*N] (local-frame lat-long BRDF, HAAR1), normals host [V][2] fp64 (theta_N, phi_N),
    vis_q [V][4**log2k] (qtree layout), light [batch][stride >= 4**log2k] (HAAR1 prefixes)
    -> radiance [V][batch] = integral of L_b * Rot(theta_v, phi_v) rho * V_v (the paper's shading:
    the BRDF rotated per normal, then the triple product)."""
    lib = load()
    _dev_f32(brdf, "brdf")
    _dev_f32(vis_q, "vis_q")
    _dev_f32(light, "light")
    log2n = _log2n_pow4(brdf.numel(), "brdf")
    nrm = np.ascontiguousarray(np.asarray(normals, dtype=np.float64))
    V = vis_q.shape[0]
    kf = 4 ** log2k
    if nrm.shape != (V, 2):
        raise ValueError("normals must be [V][2] (theta_N, phi_N)")
    if vis_q.dim() != 2 or vis_q.shape[1] != kf:
        raise ValueError("vis_q must be [V][4**log2k]")
    if light.dim() != 2 or light.shape[1] < kf:
        raise ValueError("light must be [batch][stride >= 4**log2k]")
    B, stride = light.shape
    out = _out(out, (V, B), vis_q.device)
    need = relight_brdf_rotated_workspace_bytes(log2n, log2k, B)
    workspace = _aligned_workspace(need, workspace, vis_q.device)
    st = lib.relight_vertices_brdf_rotated(brdf.data_ptr(), log2n, nrm.ctypes.data, V, vis_q.data_ptr(), log2k,
                                           light.data_ptr(), stride, B, out.data_ptr(), workspace.data_ptr(), need,
                                           _stream_ptr(stream))
    check("relight_vertices_brdf_rotated", st)
    return out


def hs_fill_sparse_transfer(indices: torch.Tensor, values: torch.Tensor, row_start: int, faces: int, log2n: int,
                            dense_levels: int, seed: int, stream: Optional[torch.cuda.Stream] = None):
    """Fill indices/values [rows][K_s] with synth.sparse_transfer_rows (bit for bit)."""
    lib = load()
    rows, ks = indices.shape
    st = lib.hs_fill_sparse_transfer(indices.data_ptr(), values.data_ptr(), row_start, rows, faces, log2n, ks,
                                     dense_levels, seed % 2**64, _stream_ptr(stream))
    check("hs_fill_sparse_transfer", st)
    return indices, values


def hs_fill_transfer(out: torch.Tensor, row_start: int, faces: int, k_face: int, seed: int, stream_id: int,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Fill out [rows][faces*k_face] with the seeded synthetic transfer rows (synth.transfer_rows)."""
    lib = load()
    _dev_f32(out, "out")
    rows = out.shape[0]
    st = lib.hs_fill_transfer(out.data_ptr(), row_start, rows, faces, k_face, seed % 2**64, stream_id % 2**64,
                              _stream_ptr(stream))
    check("hs_fill_transfer", st)
    return out


def shift_and_relight(light: torch.Tensor, shifts, transfer: torch.Tensor, faces: int, k_face: int,
                      band_levels: int, shifted: Optional[torch.Tensor] = None, radiance: Optional[torch.Tensor] = None,
                      workspace: Optional[torch.Tensor] = None, relight_workspace: Optional[torch.Tensor] = None,
                      stream: Optional[torch.cuda.Stream] = None):
    """One step of the hot path: shift every frame's pyramids in the Haar domain (band only), then
    relight every vertex with the shifted band.  Returns (shifted band, radiance)."""
    shifted = haar_shift_coeffs(light, shifts, 2, band_levels, out=shifted, workspace=workspace, stream=stream)
    radiance = relight_vertices(transfer, shifted, faces, k_face, out=radiance, workspace=relight_workspace,
                                stream=stream)
    return shifted, radiance
