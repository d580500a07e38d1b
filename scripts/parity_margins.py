"""Parity margins (not a test): relative L2 error against the fp64 oracle of every benchmarked
configuration, on the bench's inputs and launch configurations (sampled vertices where the oracle
cannot afford all of them).  Output: one line per config; the gate is 1e-5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1705_07272_b200 as hs  # noqa: E402
from oracle import relight as orelight  # noqa: E402
from oracle import shift as oshift  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


out = {}
rng = np.random.default_rng(2024)
# c2: one 32x32 map, shift (3.25, 7.5), 1k vertices
cfg = synth.config("c2")
L = synth.light_pyramids(cfg.seed, 1, 1, cfg.log2n)
sh = np.array([[[3.25, 7.5]]])
T = synth.transfer_rows(cfg.seed, 0, cfg.vertices, 1, cfg.k_face)
band = hs.haar_shift_coeffs(t(L), sh, 2)
R = hs.relight_vertices(t(T), band, 1, cfg.k_face).cpu().numpy()
out["c2 radiance"] = rel(R, orelight.relight(T, oshift.shift_coeffs(L, sh, 2), 1, cfg.k_face))
# c3: 10k vertices, frames 0, 37, 200 (1-degree azimuth steps)
cfg = synth.config("c3")
L = synth.light_pyramids(cfg.seed, 1, cfg.faces, cfg.log2n)
T = synth.transfer_rows(cfg.seed, 0, cfg.vertices, cfg.faces, cfg.k_face)
worst = 0.0
for fr in (1, 37, 200):
    sh = np.broadcast_to(synth.c3_shifts(cfg.log2n, 360)[fr][None, None, :], (1, cfg.faces, 2))
    band = hs.haar_shift_coeffs(t(L), sh, 2)
    R = hs.relight_vertices(t(T), band, cfg.faces, cfg.k_face).cpu().numpy()
    worst = max(worst, rel(R, orelight.relight(T, oshift.shift_coeffs(L, sh, 2), cfg.faces, cfg.k_face)))
out["c3 radiance (3 frames, worst)"] = worst
# c5-shaped light (64 frames of 6 x 256^2) shared by c5x / c5s / c5t
cfg5 = synth.config("c5")
B, F, n = cfg5.frames, cfg5.faces, cfg5.log2n
light_np = synth.light_pyramids(cfg5.seed, B, F, n)
sh5 = np.broadcast_to(synth.c5_shifts(cfg5.seed, B, n)[:, None, :], (B, F, 2)).copy()
full = hs.haar_shift_coeffs(t(light_np), sh5, 2)
ref_full = oshift.shift_coeffs(light_np, sh5, 2)
out["c5 shifted pyramids (64 frames, full)"] = rel(full.cpu().numpy(), ref_full)
out["c5 shifted band (levels < 5)"] = rel(full.cpu().numpy()[:, :, :1024], ref_full[:, :, :1024])
for name, kf in (("c5", 1024), ("c5x", 4096)):
    rows = rng.integers(0, 1_000_000, 96)
    T = np.concatenate([synth.transfer_rows(cfg5.seed, int(v), 1, F, kf) for v in rows])
    R = hs.relight_vertices(t(T), full, F, kf).cpu().numpy()
    out[f"{name} radiance (96 sampled vertices)"] = rel(R, orelight.relight(T, ref_full, F, kf))
# c5s: sparse K_s = 256 over the full pyramids
idx, val = synth.sparse_transfer_rows(cfg5.seed, 0, 3000, F, n, 256, 2)
R = hs.relight_vertices_sparse(torch.from_numpy(idx).cuda(), t(val), full).cpu().numpy()
out["c5s radiance (3000 vertices)"] = rel(R, orelight.relight_sparse(idx, val, ref_full.reshape(B, -1)))
# c5t: triple product on the band
rho = synth.shading_rows(cfg5.seed, 0, 2000, F, 1024, synth.STREAM_BRDF)
vis = synth.shading_rows(cfg5.seed, 0, 2000, F, 1024, synth.STREAM_VIS)
rq = hs.haar_pack_qtree(t(rho).view(2000, F, 1024), 5)
vq = hs.haar_pack_qtree(t(vis).view(2000, F, 1024), 5)
R = hs.relight_vertices_triple(rq, vq, full, F, 1024).cpu().numpy()
out["c5t radiance (2000 vertices)"] = rel(R, orelight.relight_triple(rho, vis, ref_full[:, :, :1024], F, 1024))
# c4: the full 100k-vertex job on the fused path (residue planes at N = 128), 24 sampled vertices
cfg4 = synth.config("c4")
V4, F4, n4 = cfg4.vertices, cfg4.faces, cfg4.log2n
T4 = torch.empty((V4, F4 * 4 ** n4), dtype=torch.float32, device="cuda")
hs.hs_fill_transfer(T4, 0, F4, 4 ** n4, cfg4.seed, synth.STREAM_T)
L4 = synth.light_pyramids(cfg4.seed, 1, F4, n4)[0]
sv4 = synth.c4_vertex_shifts(cfg4.seed, V4, n4)
R4 = hs.relight_vertices_shifted(T4, t(L4), t(sv4)).cpu().numpy()
del T4
rows4 = np.unique(np.concatenate([[0, V4 - 1], rng.integers(0, V4, 22)]))
ref4 = np.array([orelight.relight_shifted(synth.transfer_rows(cfg4.seed, int(v), 1, F4, 4 ** n4), L4,
                                          sv4[v:v + 1].astype(np.float64))[0] for v in rows4])
out[f"c4 radiance ({len(rows4)} sampled vertices)"] = rel(R4[rows4], ref4)
# c6r: rotation of 4096 maps of 64^2 against the chain-rule oracle, 16 sampled maps
from oracle import rotate as orot  # noqa: E402
cfg6 = synth.config("c6r")
maps6 = synth.smooth_sphere_maps(cfg6.seed, cfg6.frames, cfg6.log2n)
ang6 = synth.rotation_angles(cfg6.seed, cfg6.frames)
got6 = hs.haar_rotate_coeffs(t(maps6), ang6).cpu().numpy()
pick = rng.integers(0, cfg6.frames, 16)
out["c6r rotated maps (16 sampled, max)"] = max(rel(got6[b], orot.rotate_coeffs_chain(maps6[b], *ang6[b]))
                                                for b in pick)
# c7s: the composed shading (rows f1 + f3) on the bench's inputs, 16384 vertices, 24 sampled
# vertices against the chain-rule oracle + the pixel-domain triple integral
cfg7 = synth.config("c7s")
n7, B7, k7, kf7, V7 = cfg7.log2n, cfg7.frames, cfg7.band_levels, cfg7.k_face, cfg7.vertices
brdf7 = synth.smooth_sphere_maps(cfg7.seed, 1, n7)[0]
vis7 = synth.shading_rows(cfg7.seed, 0, V7, 1, kf7, synth.STREAM_VIS)
vq7 = hs.haar_pack_qtree(t(vis7).view(V7, 1, kf7), k7).view(V7, kf7)
rng7 = np.random.default_rng([cfg7.seed, 7])
nv7 = rng7.normal(size=(V7, 3))
nv7 /= np.linalg.norm(nv7, axis=1, keepdims=True)
nrm7 = np.stack([np.arccos(np.clip(nv7[:, 1], -1.0, 1.0)), np.mod(np.arctan2(nv7[:, 0], nv7[:, 2]), 2 * np.pi)], 1)
L7 = synth.light_pyramids(cfg7.seed, B7, 1, n7)
sh7 = np.stack([np.zeros(B7), np.arange(B7) * (1 << n7) / 64.0], axis=1)[:, None, :]
band7 = hs.haar_shift_coeffs(t(L7), sh7, 2, k7)
R7 = hs.relight_vertices_brdf_rotated(t(brdf7), nrm7, vq7, band7.view(B7, kf7), k7).cpu().numpy()
rows7 = rng.integers(0, V7, 24)
rho7 = np.stack([orot.rotate_coeffs_chain(brdf7.astype(np.float64), float(nrm7[v, 0]), float(nrm7[v, 1]))[:kf7]
                 for v in rows7])
Lb7 = oshift.shift_coeffs(L7, sh7, 2)[:, :, :kf7]
out["c7s radiance (24 sampled vertices)"] = rel(R7[rows7], orelight.relight_triple(rho7, vis7[rows7].astype(np.float64),
                                                                                  Lb7, 1, kf7))
torch.cuda.synchronize()
for k, v in out.items():
    print(f"{k:42s} {v:.3e}  ({'ok' if v <= 1e-5 else 'OVER'}; margin x{1e-5 / v:.1f})")
