"""Oracle: relight = light-transport inner product, fp64 NumPy -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py; the product path never imports this).

PAPER.md eq:tripleSum writes outgoing radiance as sum_ijk C_ijk a_i b_j c_k with
C_ijk the integral of three basis functions.  With the transfer vector T holding BRDF x
visibility projected together (PRT transfer; reading R15) the third factor is
the constant 1 = the level-0 scaling function, and the Tripling Coefficient Theorem's cases (a)
and (c) give C_{i j 0} = delta_ij in the orthonormal unit-square basis: the
triple sum collapses to the plain coefficient dot product  r = sum_k L_k T_k  ("the rotated data
is plugged in the triple integral computation").

* ``relight``:          R[v][b] = sum_f sum_{k<K_face} T[v][f K_face + k] L'[b][f][k]
* ``relight_shifted``:  r_v = < S_{s_v} L , T_v >, the shifted pyramid built per vertex by
                        inverse -> shift -> forward (shift.py); the inverse is shared.
* ``relight_triple``:   the full triple product with BRDF and visibility
                        kept separate: R[v][b] = sum_f integral of L'_b,f * rho_v,f * V_v,f, the
                        integral eq:tripleSum abbreviates, evaluated by brute force
                        on the pixels of the truncated pyramids.
"""
from __future__ import annotations

import numpy as np

from . import haar, shift

__all__ = ["relight", "relight_shifted", "relight_sparse", "relight_triple"]


def relight(transfer: np.ndarray, light: np.ndarray, faces: int, k_face: int) -> np.ndarray:
    """transfer [V][faces*k_face], light [B][faces][>= k_face] -> radiance [V][B] (fp64 BLAS)."""
    T = np.asarray(transfer, dtype=np.float64)
    L = np.asarray(light, dtype=np.float64)
    B = L.shape[0]
    band = L[:, :faces, :k_face].reshape(B, faces * k_face)
    return T @ band.T


def relight_sparse(idx: np.ndarray, val: np.ndarray, light: np.ndarray) -> np.ndarray:
    """Sparse transfer (non-linear approximation): vertex v keeps
    K_s coefficients (idx[v][k] into the concatenated per-face pyramids, val[v][k]); the double
    product is R[v][b] = sum_k val[v][k] * light[b][idx[v][k]]  (light [B][faces*N*N], fp64)."""
    L = np.asarray(light, dtype=np.float64).reshape(np.asarray(light).shape[0], -1)
    vals = np.asarray(val, dtype=np.float64)
    out = np.empty((vals.shape[0], L.shape[0]), dtype=np.float64)
    for v in range(vals.shape[0]):
        out[v] = L[:, np.asarray(idx[v], dtype=np.int64)] @ vals[v]
    return out


def relight_shifted(transfer: np.ndarray, light: np.ndarray, vertex_shifts: np.ndarray) -> np.ndarray:
    """transfer [V][faces*N*N], light [faces][N*N] (one full pyramid per face), vertex_shifts
    [V][2] (sy, sx), the same shift for every face of a vertex -> radiance [V] (fp64)."""
    T = np.asarray(transfer, dtype=np.float64)
    L = np.asarray(light, dtype=np.float64)
    F, K = L.shape
    pixels = [haar.inverse2d(L[f]) for f in range(F)]          # inverse once (shared by vertices)
    out = np.empty(T.shape[0], dtype=np.float64)
    for v in range(T.shape[0]):
        sy, sx = float(vertex_shifts[v][0]), float(vertex_shifts[v][1])
        acc = 0.0
        for f in range(F):
            shifted = haar.forward2d(shift.shift_pixels2d(pixels[f], sy, sx))
            acc += float(np.dot(shifted, T[v, f * K:(f + 1) * K]))
        out[v] = acc
    return out


def _cells(prefix_rows: np.ndarray, k: int) -> np.ndarray:
    """[rows][4**k] HAAR1 prefixes (levels < k) -> [rows][4**k] cell values of the 2**k x 2**k
    piecewise-constant functions they represent (the prefix is itself a complete level-k pyramid
    in the unit-square normalisation, R1)."""
    rows = np.asarray(prefix_rows, dtype=np.float64)
    return np.stack([haar.inverse2d(r).reshape(-1) for r in rows]) if rows.shape[0] else rows.copy()


def relight_triple(brdf: np.ndarray, vis: np.ndarray, light: np.ndarray, faces: int, k_face: int) -> np.ndarray:
    """brdf, vis [V][faces*k_face] (HAAR1 prefixes, k_face = 4**k), light [B][faces][>= k_face]
    -> radiance [V][B], fp64:

        R[v][b] = sum_f  integral over the unit square of  L_bf * rho_vf * V_vf
                = sum_f  mean over the 4**k cells of the product of the three reconstructions.

    This is the triple integral of eq:tripleSum before it is expanded into the sum
    sum_ijk C_ijk a_i b_j c_k; the tests pin it to that sum with C_ijk integrated from the basis
    table, and to the Tripling Coefficient Theorem's cases."""
    k = int(round(np.log2(k_face) / 2))
    if 4 ** k != k_face:
        raise ValueError("k_face must be a power of 4")
    rho = np.asarray(brdf, dtype=np.float64)
    vv = np.asarray(vis, dtype=np.float64)
    L = np.asarray(light, dtype=np.float64)
    V, B = rho.shape[0], L.shape[0]
    out = np.zeros((V, B), dtype=np.float64)
    for f in range(faces):
        sl = slice(f * k_face, (f + 1) * k_face)
        prod = _cells(rho[:, sl], k) * _cells(vv[:, sl], k)          # [V][cells]
        lc = _cells(L[:, f, :k_face], k)                              # [B][cells]
        out += prod @ lc.T / k_face
    return out
