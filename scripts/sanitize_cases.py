"""Small invocations of every kernel in libhaarshift.so, for compute-sanitizer (memcheck /
racecheck / synccheck).  Prints max relative errors against the oracle so a sanitizer run also
checks results."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1705_07272_b200 as hs  # noqa: E402
from oracle import relight as orelight  # noqa: E402
from oracle import shift as oshift  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


errs = {}
# 1D and 2D shifts incl. dyadic, identity, band, chunked, large-face (global coarse) paths
c = synth.random_signals(1, 6, 64)[:, None, :]
s = np.array([0.0, 3.0, 32.0, 0.5, -7.25, 16.0])[:, None, None]
errs["shift1d"] = rel(hs.haar_shift_coeffs(t(c), s, 1).cpu().numpy(), oshift.shift_coeffs(c, s, 1))
for n in (2, 5, 8):
    L = synth.light_pyramids(2, 3, 2, n)
    sh = np.array([[[1.5, -2.25], [0, 0]], [[2 ** n / 2, 2 ** n / 4], [3, 5]], [[0.1, 0.9], [7.5, 0]]])
    errs[f"shift2d_n{n}"] = rel(hs.haar_shift_coeffs(t(L), sh, 2).cpu().numpy(), oshift.shift_coeffs(L, sh, 2))
    errs[f"shift2d_band_n{n}"] = rel(hs.haar_shift_coeffs(t(L), sh, 2, band_levels=2).cpu().numpy(),
                                    oshift.shift_coeffs(L, sh, 2, band_levels=2))
L = synth.light_pyramids(3, 1, 1, 10)
sh = np.array([[[11.25, -3.5]]])
errs["shift2d_n10"] = rel(hs.haar_shift_coeffs(t(L), sh, 2).cpu().numpy(), oshift.shift_coeffs(L, sh, 2))
# relight: GEMV, CUDA-core GEMM, tcgen05 GEMM (with a row tail)
for B in (1, 5, 13, 64):
    T = synth.transfer_rows(4, 0, 333, 6, 256)
    Lb = synth.light_pyramids(5, B, 6, 4)
    errs[f"relight_b{B}"] = rel(hs.relight_vertices(t(T), t(Lb), 6, 256).cpu().numpy(), orelight.relight(T, Lb, 6, 256))
# fused per-vertex relight (fused N <= 128 path and the chunked N = 256 path)
for n, V in ((5, 37), (8, 3)):
    Lf = synth.light_pyramids(6, 1, 6, n)[0]
    T = synth.transfer_rows(7, 0, V, 6, 4 ** n)
    sv = synth.c4_vertex_shifts(8, V, n)
    errs[f"relight_shifted_n{n}"] = rel(hs.relight_vertices_shifted(t(T), t(Lf), t(sv)).cpu().numpy(),
                                        orelight.relight_shifted(T, Lf, sv.astype(np.float64)))
out = torch.empty((9, 6 * 16), device="cuda")
hs.hs_fill_transfer(out, 5, 6, 16, 9, synth.STREAM_T)
errs["fill"] = float(np.abs(out.cpu().numpy() - synth.transfer_rows(9, 5, 9, 6, 16)).max())
# widened rows: coarse start (f4), sparse (f2), triple product (f3, both paths), rotation (f1, exact parts)
Lc = synth.light_pyramids(10, 2, 2, 6)
shc = np.array([[[8.0, -4.0], [12.0, 20.0]], [[4.0, 4.0], [0.0, 8.0]]])      # multiples of 2^(n-L): exact
errs["coarse_L4"] = rel(hs.haar_shift_coeffs_coarse(t(Lc), shc, 4).cpu().numpy(),
                        oshift.shift_coeffs(Lc, shc, 2, band_levels=4))
idx, val = synth.sparse_transfer_rows(11, 0, 57, 2, 5, 40)
Ls = synth.light_pyramids(12, 3, 2, 5)
errs["sparse_b3"] = rel(hs.relight_vertices_sparse(torch.from_numpy(idx).cuda(), t(val), t(Ls)).cpu().numpy(),
                        orelight.relight_sparse(idx, val, Ls.reshape(3, -1)))
for B in (3, 64):
    rho = synth.shading_rows(13, 0, 131, 2, 64, synth.STREAM_BRDF)
    vis = synth.shading_rows(13, 0, 131, 2, 64, synth.STREAM_VIS)
    Lt = synth.light_pyramids(14, B, 2, 3)
    rq = hs.haar_pack_qtree(t(rho).view(131, 2, 64), 3)
    vq = hs.haar_pack_qtree(t(vis).view(131, 2, 64), 3)
    errs[f"triple_b{B}"] = rel(hs.relight_vertices_triple(rq, vq, t(Lt), 2, 64).cpu().numpy(),
                               orelight.relight_triple(rho, vis, Lt, 2, 64))
from oracle import rotate as orot  # noqa: E402
cm = synth.smooth_sphere_maps(15, 3, 4)
ang = np.array([[0.0, 0.0], [0.0, 2 * np.pi * 3 / 16], [0.0, -2 * np.pi / 16]])
got = hs.haar_rotate_coeffs(t(cm), ang).cpu().numpy()
errs["rotate_exact"] = max(rel(got[b], orot.rotate_coeffs(cm[b].astype(np.float64), *ang[b])) for b in range(3))
got = hs.haar_rotate_coeffs(t(cm), np.array([[0.7, 1.0], [-0.4, 0.2], [1.2, 3.0]])).cpu().numpy()
errs["rotate_finite"] = 0.0 if np.isfinite(got).all() else 1.0
torch.cuda.synchronize()
for k, v in errs.items():
    print(f"{k}: {v:.3e}")
bad = {k: v for k, v in errs.items() if not (v <= 1e-5)}
print("FAIL" if bad else "ALL OK", bad)
sys.exit(1 if bad else 0)
