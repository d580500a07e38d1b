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

``rotate_coeffs_chain`` is the paper's own algorithm, step by step (P:405-459 chain rule on the
difference fields, P:466-497 the [1,1] x [1,2,1] recursion, P:459/P:508 the azimuth shift), with
the readings R25-R27 of DESIGN.md where the paper is silent or garbled.  The method is first order
in the pixel size, so it approximates the spatial rotation above; the GPU is held to
``rotate_coeffs_chain`` at 1e-5, and ``rotate_coeffs_chain`` is pinned to the spatial rotation by
its exact cases (alpha = 0, alpha = pi, constants, pure azimuth) and by its convergence with N
(tests/test_oracle_rotate.py).
"""
from __future__ import annotations

import numpy as np

from . import haar, shift

__all__ = ["rotated_angles", "elevate_pixels", "rotate_coeffs", "chain_rule_fields", "periodic_closure",
           "fields_bottom_up", "rotated_dc", "rotate_coeffs_chain", "psnr"]


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


def _fields_of_pixels(f: np.ndarray):
    """Difference fields of the pixel map at the finest level (eq:pde1-2's X, Y):
    X[r][c] = f[r][c] - f[r][c+1] (periodic in phi), Y[r][c] = f[r][c] - f[r+1][c] for r < N-1,
    plus the rows across the poles (R26): the row beyond a pole is the pole row seen from
    phi + pi, so X[-1][c] = X[0][c + N/2], X[N][c] = X[N-1][c + N/2], Y[-1][c] = f[0][c+N/2] - f[0][c],
    Y[N-1][c] = f[N-1][c] - f[N-1][c+N/2].  Returned with the extra rows: Xe rows -1..N (N+2 rows),
    Ye rows -1..N-1 (N+1 rows)."""
    N = f.shape[0]
    h = N // 2
    X = f - np.roll(f, -1, axis=1)
    Y = f[:-1] - f[1:]
    Xe = np.vstack([np.roll(X[0], -h)[None], X, np.roll(X[N - 1], -h)[None]])
    Ye = np.vstack([(np.roll(f[0], -h) - f[0])[None], Y, (f[N - 1] - np.roll(f[N - 1], -h))[None]])
    return Xe, Ye


def _bilinear_rows(P: np.ndarray, y: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Bilinear sample of a field plane P whose row k sits at index y = k - 1 (P's first row is the
    row across the top pole), index coordinates (y, x), periodic in x."""
    N = P.shape[1]
    y0 = np.floor(y).astype(np.int64)
    x0 = np.floor(x).astype(np.int64)
    wy = y - y0
    wx = x - x0
    r0 = np.clip(y0 + 1, 0, P.shape[0] - 1)
    r1 = np.clip(y0 + 2, 0, P.shape[0] - 1)
    c0 = np.mod(x0, N)
    c1 = np.mod(x0 + 1, N)
    return ((1 - wy) * ((1 - wx) * P[r0, c0] + wx * P[r0, c1]) +
            wy * ((1 - wx) * P[r1, c0] + wx * P[r1, c1]))


def _cell_means(f: np.ndarray, M: int) -> np.ndarray:
    N = f.shape[0]
    k = N // M
    return f.reshape(M, k, M, k).mean(axis=(1, 3))


def chain_rule_fields(f: np.ndarray, alpha: float):
    """Step 2 of ``rotate_coeffs_chain``: the chain rule (eq:pde1-2; Fig. 4)
    per output difference X_g[i][j] = g(i, j) - g(i, j+1) and Y_g[i][j] = g(i, j) - g(i+1, j),
    g(theta, phi) = f(Theta, Phi), from the difference fields of the pixel map f (step 1, R26).
    With (Theta0, Phi0), (Theta1, Phi1) the rotated endpoints and (ThetaM, PhiM) the rotated
    midpoint, dTheta = Theta0 - Theta1, dPhi = Phi0 - Phi1 wrapped to (-pi, pi], f_Theta = -Y_f /
    dtheta and f_Phi = -X_f / dphi interpolated bilinearly at the midpoint (X_f sits at
    (r, c + 1/2), Y_f at (r + 1/2, c) in pixel-centre coordinates):
    D = f_Theta dTheta + f_Phi dPhi  (R26: increments of the two samples, not derivatives).
    Returns the raw (X_g, Y_g), N x N each."""
    N = f.shape[0]
    Xe, Ye = _fields_of_pixels(f)
    dth, dph = np.pi / N, 2.0 * np.pi / N
    I, J = np.meshgrid(np.arange(N, dtype=np.float64), np.arange(N, dtype=np.float64), indexing="ij")
    T0, P0 = rotated_angles((I + 0.5) * dth, (J + 0.5) * dph, alpha)
    out_fields = []
    for di, dj in ((0.0, 1.0), (1.0, 0.0)):            # X_g (neighbour in phi), Y_g (in theta)
        T1, P1 = rotated_angles((I + 0.5 + di) * dth, (J + 0.5 + dj) * dph, alpha)
        TM, PM = rotated_angles((I + 0.5 + 0.5 * di) * dth, (J + 0.5 + 0.5 * dj) * dph, alpha)
        y = TM / dth - 0.5                             # pixel-centre coordinates of the midpoint
        x = PM / dph - 0.5
        xf = _bilinear_rows(Xe, y, x - 0.5)
        yf = _bilinear_rows(Ye, y - 0.5, x)
        dT = T0 - T1
        dP = P0 - P1
        dP = np.where(dP > np.pi, dP - 2 * np.pi, np.where(dP < -np.pi, dP + 2 * np.pi, dP))
        out_fields.append(-yf * dT / dth - xf * dP / dph)
    return out_fields[0], out_fields[1]


def periodic_closure(Xg: np.ndarray) -> np.ndarray:
    """Step 3 (R27): the exact X field of any periodic N x N map sums to 0 along every row
    (a telescoping sum of periodic differences); the chain rule's does not, so each row of X_g
    loses its mean -- the orthogonal projection onto the fields that can be differences of a map.
    (Y_g needs no closure: its last row feeds only the level-0 residual of the recursion, never
    an output coefficient -- pinned in tests/test_oracle_rotate.py.)"""
    return Xg - Xg.mean(axis=1, keepdims=True)


def fields_bottom_up(Xg: np.ndarray, Yg: np.ndarray):
    """Steps 4-5: Z_g[i][j] = X_g[i][j] - X_g[i+1][j] (R27) and the recursion
    h_s = [1,1], h_t = [1,2,1], decimated by 2 (eq:conv-sker P:466-478):
    X_l = 1/4 (h_s along theta) (h_t along phi) X_{l+1} at even positions, Y_l the transpose,
    Z_l = 1/4 h_t x h_t; the level-l details H = 1/4 (X[2i][2j] + X[2i+1][2j]),
    V = 1/4 (Y[2i][2j] + Y[2i][2j+1]), D = 1/4 Z[2i][2j], times 2**-l (unit-square scale).
    Returns (details[0..n-1] as (H, V, D), the level-0 residuals (X_0, Y_0, Z_0))."""
    N = Xg.shape[0]
    n = haar.log2_exact(N)
    details = [None] * n
    X, Y, Z = Xg, Yg, Xg - np.roll(Xg, -1, axis=0)
    for l in range(n - 1, -1, -1):
        s = 2.0 ** (-l)
        H = 0.25 * (X[0::2, 0::2] + X[1::2, 0::2]) * s
        V = 0.25 * (Y[0::2, 0::2] + Y[0::2, 1::2]) * s
        D = 0.25 * Z[0::2, 0::2] * s
        details[l] = (H, V, D)

        def ht(A, axis):                               # [1, 2, 1] centred on the even sample
            return A + 2.0 * np.roll(A, -1, axis=axis) + np.roll(A, -2, axis=axis)

        def hs(A, axis):                               # [1, 1]
            return A + np.roll(A, -1, axis=axis)
        X = 0.25 * ht(hs(X, 0), 1)[0::2, 0::2]
        Y = 0.25 * hs(ht(Y, 0), 1)[0::2, 0::2]
        Z = 0.25 * ht(ht(Z, 0), 1)[0::2, 0::2]
    return details, (float(X[0, 0]), float(Y[0, 0]), float(Z[0, 0]))


DC_LEVEL = 6   # R27: the scaling coefficient comes from the level-min(n, 6) approximation


def rotated_dc(f: np.ndarray, alpha: float) -> float:
    """Step 6 (R27): the mean over the N x N grid of the level-min(n, DC_LEVEL) cell means
    of f sampled bilinearly at the rotated pixel centres (poles reflected, phi periodic)."""
    N = f.shape[0]
    n = haar.log2_exact(N)
    M = 1 << min(n, DC_LEVEL)
    A = _cell_means(f, M)
    dth, dph = np.pi / N, 2.0 * np.pi / N
    I, J = np.meshgrid(np.arange(N, dtype=np.float64), np.arange(N, dtype=np.float64), indexing="ij")
    T0, P0 = rotated_angles((I + 0.5) * dth, (J + 0.5) * dph, alpha)
    y = T0 * M / np.pi - 0.5
    x = P0 * M / (2.0 * np.pi) - 0.5
    y0 = np.floor(y).astype(np.int64)
    x0 = np.floor(x).astype(np.int64)
    wy, wx = y - y0, x - x0
    dc = np.zeros_like(y)
    for dy, wyv in ((0, 1 - wy), (1, wy)):
        for dx, wxv in ((0, 1 - wx), (1, wx)):
            r = y0 + dy
            cc = x0 + dx
            top, bot = r < 0, r >= M
            r = np.where(top, -1 - r, np.where(bot, 2 * M - 1 - r, r))
            cc = np.where(top | bot, cc + M // 2, cc)
            dc += wyv * wxv * A[r, np.mod(cc, M)]
    return float(dc.mean())


def rotate_coeffs_chain(c: np.ndarray, alpha: float, beta: float) -> np.ndarray:
    """The paper's Haar-domain rotation of one N x N lat-long map (HAAR1 in, HAAR1 out), fp64:

    1. the difference fields X_f, Y_f of f at the finest level with the rows across the poles (R26);
    2. the chain rule per output difference (``chain_rule_fields``);
    3. the periodic closure of X_g (``periodic_closure``, R27);
    4-5. Z_g and the [1,1] x [1,2,1] recursion to every detail level (``fields_bottom_up``);
    6. the scaling coefficient (``rotated_dc``, R27);
    7. the azimuth: the exact shift by beta N / (2 pi) columns."""
    f = haar.inverse2d(np.asarray(c, dtype=np.float64))
    N = f.shape[0]
    Xg, Yg = chain_rule_fields(f, alpha)
    Xg = periodic_closure(Xg)
    details, _ = fields_bottom_up(Xg, Yg)
    coeffs = haar.pack2d(rotated_dc(f, alpha), details)
    return shift.shift_coeffs2d(coeffs, 0.0, beta * N / (2.0 * np.pi))


def psnr(test_coeffs: np.ndarray, ref_coeffs: np.ndarray) -> float:
    """PSNR in dB between the pixel maps of two pyramids, peak = max |reference pixel|."""
    a = haar.inverse2d(np.asarray(test_coeffs, dtype=np.float64))
    b = haar.inverse2d(np.asarray(ref_coeffs, dtype=np.float64))
    mse = float(np.mean((a - b) ** 2))
    peak = float(np.max(np.abs(b)))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(peak * peak / mse)
