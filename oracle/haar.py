"""Oracle: Haar transforms and HAAR1 packing, fp64 NumPy -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py; the product path never imports this).

Conventions (DESIGN.md §2 readings R1, R2):

* 2D: unit-square orthonormal non-separable Haar: the level-l wavelet is +-2**l on
  its square of side 2**-l, a coefficient is the integral over the unit square of f * psi (for a
  pixel map, the mean over pixels of f * psi), the scaling coefficient is the mean.  Signs
  (SPEC.md S:78): horizontal + on the left half, vertical + on the top half, diagonal + on the
  main-diagonal quadrants.  Rows index theta (top first), columns phi.
* 1D: unit-interval orthonormal Haar: the level-l wavelet is +-2**(l/2) on an interval of length
  2**-l, + on the left half.
* HAAR1 order: scaling, then per level ascending, per type (H, V, D), row-major.
  2D index(l, t, i, j) = 4**l * (1 + t) + i * 2**l + j; 1D index(l, k) = 2**l + k.

The transforms are written as the textbook quadtree recursion on quadrant means ("averaging"
details), then scaled to the unit-square normalisation: a level-l unit-square coefficient is
2**-l (2D) or 2**(-l/2) (1D) times the averaging detail.
"""
from __future__ import annotations

import numpy as np

__all__ = ["forward2d", "inverse2d", "forward1d", "inverse1d", "pack2d", "unpack2d", "pack1d",
           "unpack1d", "log2_exact"]


def log2_exact(N: int) -> int:
    n = int(N).bit_length() - 1
    if N < 1 or (1 << n) != N:
        raise ValueError(f"size {N} is not a power of two (SPEC.md S:46)")
    return n


# ------------------------------------------------------------------------------------ packing

def pack2d(scaling: float, details: list) -> np.ndarray:
    """details[l] = (H_l, V_l, D_l), each 2**l x 2**l (unit-square) -> HAAR1 vector of N*N."""
    n = len(details)
    out = np.zeros(4 ** n, dtype=np.float64)
    out[0] = scaling
    for l, (H, V, D) in enumerate(details):
        base = 4 ** l
        out[base * 1:base * 2] = np.asarray(H, dtype=np.float64).reshape(-1)
        out[base * 2:base * 3] = np.asarray(V, dtype=np.float64).reshape(-1)
        out[base * 3:base * 4] = np.asarray(D, dtype=np.float64).reshape(-1)
    return out


def unpack2d(c: np.ndarray):
    """HAAR1 vector of N*N -> (scaling, [(H_l, V_l, D_l)]) in fp64."""
    c = np.asarray(c, dtype=np.float64).reshape(-1)
    n = log2_exact(int(round(np.sqrt(c.size))))
    if 4 ** n != c.size:
        raise ValueError("HAAR1 2D vector length must be 4**n")
    details = []
    for l in range(n):
        g = 1 << l
        base = 4 ** l
        details.append(tuple(c[base * (1 + t):base * (2 + t)].reshape(g, g) for t in range(3)))
    return float(c[0]), details


def pack1d(scaling: float, details: list) -> np.ndarray:
    n = len(details)
    out = np.zeros(2 ** n, dtype=np.float64)
    out[0] = scaling
    for l, d in enumerate(details):
        out[2 ** l:2 ** (l + 1)] = np.asarray(d, dtype=np.float64)
    return out


def unpack1d(c: np.ndarray):
    c = np.asarray(c, dtype=np.float64).reshape(-1)
    n = log2_exact(c.size)
    return float(c[0]), [c[2 ** l:2 ** (l + 1)].copy() for l in range(n)]


# ------------------------------------------------------------------------------------ 2D

def forward2d(f: np.ndarray) -> np.ndarray:
    """Pixel map f (N x N) -> HAAR1 unit-square coefficients.

    Quadtree recursion, finest level first.  Children of cell (i, j) at level l are
    c_ab = A_{l+1}[2i+a][2j+b] (a = row offset, b = column offset):
      A_l = (c00 + c01 + c10 + c11) / 4
      H^_l = (c00 - c01 + c10 - c11) / 4      (+ left half)
      V^_l = (c00 + c01 - c10 - c11) / 4      (+ top half)
      D^_l = (c00 - c01 - c10 + c11) / 4      (+ main diagonal)
    unit-square coefficient = 2**-l * averaging detail.
    """
    A = np.asarray(f, dtype=np.float64)
    N = A.shape[0]
    if A.shape != (N, N):
        raise ValueError("map must be square")
    n = log2_exact(N)
    details = [None] * n
    for l in range(n - 1, -1, -1):
        c00 = A[0::2, 0::2]
        c01 = A[0::2, 1::2]
        c10 = A[1::2, 0::2]
        c11 = A[1::2, 1::2]
        H = (c00 - c01 + c10 - c11) / 4.0
        V = (c00 + c01 - c10 - c11) / 4.0
        D = (c00 - c01 - c10 + c11) / 4.0
        details[l] = (H * 2.0 ** -l, V * 2.0 ** -l, D * 2.0 ** -l)
        A = (c00 + c01 + c10 + c11) / 4.0
    return pack2d(float(A[0, 0]), details)


def inverse2d(c: np.ndarray) -> np.ndarray:
    """HAAR1 unit-square coefficients -> pixel map.

    Top-down from A_0 = scaling; children of (i, j): A_{l+1}[2i+a][2j+b] = A_l[i][j] + delta_ab
    with (averaging details H^, V^, D^ = 2**l * unit-square):
      delta_00 =  H^ + V^ + D^     delta_01 = -H^ + V^ - D^
      delta_10 =  H^ - V^ - D^     delta_11 = -H^ - V^ + D^
    """
    s, details = unpack2d(c)
    A = np.array([[s]], dtype=np.float64)
    for l, (H, V, D) in enumerate(details):
        Hh, Vh, Dh = H * 2.0 ** l, V * 2.0 ** l, D * 2.0 ** l
        g = 1 << l
        nxt = np.empty((2 * g, 2 * g), dtype=np.float64)
        nxt[0::2, 0::2] = A + Hh + Vh + Dh
        nxt[0::2, 1::2] = A - Hh + Vh - Dh
        nxt[1::2, 0::2] = A + Hh - Vh - Dh
        nxt[1::2, 1::2] = A - Hh - Vh + Dh
        A = nxt
    return A


# ------------------------------------------------------------------------------------ 1D

def forward1d(f: np.ndarray) -> np.ndarray:
    """Signal f (N) -> HAAR1 1D unit-interval coefficients.

    a_l[k] = (a_{l+1}[2k] + a_{l+1}[2k+1]) / 2, d^_l[k] = (a_{l+1}[2k] - a_{l+1}[2k+1]) / 2,
    unit-interval coefficient = 2**(-l/2) * d^_l.
    """
    a = np.asarray(f, dtype=np.float64).reshape(-1)
    n = log2_exact(a.size)
    details = [None] * n
    for l in range(n - 1, -1, -1):
        d = (a[0::2] - a[1::2]) / 2.0
        details[l] = d * 2.0 ** (-l / 2.0)
        a = (a[0::2] + a[1::2]) / 2.0
    return pack1d(float(a[0]), details)


def inverse1d(c: np.ndarray) -> np.ndarray:
    """a_{l+1}[2k] = a_l[k] + d^_l[k], a_{l+1}[2k+1] = a_l[k] - d^_l[k]."""
    s, details = unpack1d(c)
    a = np.array([s], dtype=np.float64)
    for l, d in enumerate(details):
        dh = d * 2.0 ** (l / 2.0)
        nxt = np.empty(2 * a.size, dtype=np.float64)
        nxt[0::2] = a + dh
        nxt[1::2] = a - dh
        a = nxt
    return a
