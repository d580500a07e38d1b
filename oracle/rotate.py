"""Oracle: rotation of lat-long maps, fp64 NumPy -- TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py; the product path never imports this).

The paper's ground truth for its Haar-domain rotation is "rotating it in the spatial domain"
(PAPER.md P:535); SPEC.md S:191-199 (rotate_map_spatial) writes that procedure out.  Here:

* lat-long map of N x N pixels: row r at theta_r = (r + 1/2) pi / N (top first), column c at
  phi_c = (c + 1/2) 2 pi / N (p = (sin t sin f, cos t, sin t cos f), Y up);
* ``rotated_angles``: the elevation rotation about X, p' = R_x(alpha) p with the active matrix
  R_x = [[1,0,0],[0,cos a,-sin a],[0,sin a,cos a]], Theta = acos(R_2 p),
  Phi = atan2(R_1 p, R_3 p) mod 2 pi (eq:theta / eq:phi);
* ``elevate_pixels``: g(r, c) = f(Theta, Phi) sampled bilinearly at the continuous pixel position
  of (Theta, Phi), periodic in phi, reflected across the poles (row -1 - k / 2N - 1 - k with the
  column moved by N / 2) -- SPEC.md S:197;
* ``rotate_coeffs``: inverse Haar -> elevate by alpha -> the exact pixel shift along phi by
  beta N / (2 pi) columns (the azimuth part "simply becomes a linear shift") ->
  forward Haar.

The GPU computes the elevation by the paper's chain rule on the coefficients' difference fields
(P:405-459), which approximates this; their agreement is reported as PSNR (R25), not
held to 1e-5.  This oracle itself is pinned in tests/test_oracle_rotate.py.
"""
from __future__ import annotations

import numpy as np

from . import haar, shift

__all__ = ["rotated_angles", "elevate_pixels", "rotate_coeffs", "psnr"]


def rotated_angles(theta, phi, alpha: float):
    """(Theta, Phi) of R_x(alpha) p(theta, phi); Phi in [0, 2 pi)."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    x = np.sin(theta) * np.sin(phi)
    y = np.cos(theta)
    z = np.sin(theta) * np.cos(phi)
    ca, sa = np.cos(alpha), np.sin(alpha)
    yr = ca * y - sa * z
    zr = sa * y + ca * z
    Th = np.arccos(np.clip(yr, -1.0, 1.0))
    Ph = np.mod(np.arctan2(x, zr), 2.0 * np.pi)
    return Th, Ph


def _sample_bilinear(f: np.ndarray, ry: np.ndarray, rx: np.ndarray) -> np.ndarray:
    """Bilinear sample of the pixel map at continuous pixel coordinates (pixel centres at
    integers), periodic in x, reflected across the poles in y."""
    N = f.shape[0]
    y0 = np.floor(ry).astype(np.int64)
    x0 = np.floor(rx).astype(np.int64)
    wy = ry - y0
    wx = rx - x0
    out = np.zeros(ry.shape)
    for dy, wyv in ((0, 1.0 - wy), (1, wy)):
        for dx, wxv in ((0, 1.0 - wx), (1, wx)):
            r = y0 + dy
            c = x0 + dx
            top = r < 0
            bot = r >= N
            r = np.where(top, -1 - r, np.where(bot, 2 * N - 1 - r, r))
            c = np.where(top | bot, c + N // 2, c)
            out += wyv * wxv * f[r, np.mod(c, N)]
    return out


def elevate_pixels(f: np.ndarray, alpha: float) -> np.ndarray:
    """g(r, c) = f(Theta(theta_r, phi_c), Phi(theta_r, phi_c)) by bilinear resampling."""
    f = np.asarray(f, dtype=np.float64)
    N = f.shape[0]
    th = (np.arange(N) + 0.5) * np.pi / N
    ph = (np.arange(N) + 0.5) * 2.0 * np.pi / N
    T, P = np.meshgrid(th, ph, indexing="ij")
    Th, Ph = rotated_angles(T, P, alpha)
    return _sample_bilinear(f, Th * N / np.pi - 0.5, Ph * N / (2.0 * np.pi) - 0.5)


def rotate_coeffs(c: np.ndarray, alpha: float, beta: float) -> np.ndarray:
    """HAAR1 pyramid of an N x N lat-long map -> the pyramid of the map elevated by alpha and
    then shifted by beta along phi (beta N / 2 pi columns, f'(x) = f(x - s), box projection)."""
    pix = haar.inverse2d(np.asarray(c, dtype=np.float64))
    N = pix.shape[0]
    g = elevate_pixels(pix, alpha)
    g = shift.shift_pixels2d(g, 0.0, beta * N / (2.0 * np.pi))
    return haar.forward2d(g)


def psnr(test_coeffs: np.ndarray, ref_coeffs: np.ndarray) -> float:
    """PSNR in dB between the pixel maps of two pyramids, peak = max |reference pixel|."""
    a = haar.inverse2d(np.asarray(test_coeffs, dtype=np.float64))
    b = haar.inverse2d(np.asarray(ref_coeffs, dtype=np.float64))
    mse = float(np.mean((a - b) ** 2))
    peak = float(np.max(np.abs(b)))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(peak * peak / mse)
