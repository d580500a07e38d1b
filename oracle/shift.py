"""Oracle: shifted Haar pyramids by inverse -> pixel-domain shift -> forward, fp64 NumPy --
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py; the product path never imports this).

This is the paper's own ground-truth procedure ("we processed the BRDF data by
rotating it in the spatial domain to generate the ground truth") applied to the azimuth/"linear
shift" part of the rotation ("a rotation with respect to the azimuth angle ...
simply becomes a linear shift"; "a simple shifting along the phi-axis").

Readings:

* R3  both axes periodic, each face an independent N x N signal (cube faces are compressed
      separately);
* R4  a fractional shift is the box projection P_{V_n} T_s: translate the piecewise-constant
      function the coefficients represent by s pixels and re-project it onto the same pixels;
* R5  s is in finest-pixel units, f'[x] = f[x - s] (content moves to higher index); shift order
      (sy, sx) = (rows/theta, columns/phi);
* R8  the scaling coefficient is whatever the forward transform gives (it is preserved exactly).
"""
from __future__ import annotations

import math

import numpy as np

from . import haar

__all__ = ["split_shift", "shift_pixels1d", "shift_pixels2d", "shift_coeffs1d", "shift_coeffs2d",
           "shift_coeffs"]


def split_shift(s: float, N: int):
    """s -> (q, phi): s reduced mod N in fp64, q = floor(s) in [0, N), phi = s - q in [0, 1)."""
    s = math.fmod(float(s), float(N))
    if s < 0.0:
        s += float(N)
    q = math.floor(s)
    phi = s - q
    if q >= N:          # s within one ulp below N after the reduction
        q -= N
    return int(q), float(phi)


def _box_project_axis(f: np.ndarray, s: float, axis: int) -> np.ndarray:
    """f'[x] = integral over pixel x of the piecewise-constant f translated by s (R4).

    Pixel x covers [x, x+1); the translated function there is f(y - s) with y - s in
    [x - q - phi, x - q + 1 - phi): it overlaps source pixel x - q - 1 over length phi and source
    pixel x - q over length 1 - phi, hence f'[x] = (1 - phi) f[x - q] + phi f[x - q - 1]
    (np.roll(f, k)[x] = f[x - k], periodic).
    """
    N = f.shape[axis]
    q, phi = split_shift(s, N)
    return (1.0 - phi) * np.roll(f, q, axis=axis) + phi * np.roll(f, q + 1, axis=axis)


def shift_pixels1d(f: np.ndarray, s: float) -> np.ndarray:
    return _box_project_axis(np.asarray(f, dtype=np.float64), s, 0)


def shift_pixels2d(f: np.ndarray, sy: float, sx: float) -> np.ndarray:
    """Separable box projection: rows by sy, then columns by sx (the two commute)."""
    g = _box_project_axis(np.asarray(f, dtype=np.float64), sy, 0)
    return _box_project_axis(g, sx, 1)


def shift_coeffs1d(c: np.ndarray, s: float) -> np.ndarray:
    """inverse -> pixel shift -> forward (1D)."""
    return haar.forward1d(shift_pixels1d(haar.inverse1d(c), s))


def shift_coeffs2d(c: np.ndarray, sy: float, sx: float) -> np.ndarray:
    """inverse -> pixel shift -> forward (2D, one face)."""
    return haar.forward2d(shift_pixels2d(haar.inverse2d(c), sy, sx))


def shift_coeffs_coarse2d(c: np.ndarray, start_level: int, sy: float, sx: float) -> np.ndarray:
    """Coarse start ("one can start at any resolution level that is lower than n-1 ...
    the computational complexity is reduced to O(N/4^k)"), reading R23: the shift of the
    level-L approximation.  Keep the HAAR1 prefix of levels < L (4**L coefficients), synthesise it
    at 2**L x 2**L (each cell the mean of its 2**(n-L) x 2**(n-L) pixels), box-project-shift that
    map by s / 2**(n-L) cells, forward transform.  Returns the 4**L coefficients (levels < L)."""
    c = np.asarray(c, dtype=np.float64).reshape(-1)
    n = haar.log2_exact(int(round(np.sqrt(c.size))))
    k = n - start_level
    prefix = c[: 4 ** start_level]
    return shift_coeffs2d(prefix, sy / 2.0 ** k, sx / 2.0 ** k)


def shift_coeffs(coeffs: np.ndarray, shifts: np.ndarray, ndim: int, band_levels: int | None = None):
    """Batched: coeffs [batch][faces][N**ndim... flattened], shifts [batch][faces][ndim] ->
    shifted pyramids (fp64), optionally truncated to the HAAR1 prefix holding the scaling and
    levels < band_levels (4**band_levels coefficients in 2D, 2**band_levels in 1D)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    shifts = np.asarray(shifts, dtype=np.float64)
    B, F, K = coeffs.shape
    out = np.empty_like(coeffs)
    for b in range(B):
        for f in range(F):
            if ndim == 2:
                out[b, f] = shift_coeffs2d(coeffs[b, f], shifts[b, f, 0], shifts[b, f, 1])
            else:
                out[b, f] = shift_coeffs1d(coeffs[b, f], shifts[b, f, 0])
    if band_levels is not None:
        out = out[:, :, :(4 if ndim == 2 else 2) ** band_levels]
    return out
