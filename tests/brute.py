"""Independent brute-force checkers used to PIN the oracle (tests only).

Nothing here imports ``oracle``: every routine is built from the definitions of the basis and of
the shift, in the most literal (slow) way, so that a plausible mistake in the oracle (a dropped
term, a wrong sign or index, a transposed operand, a wrong normalisation) disagrees with them.

* ``basis2d(n)`` / ``basis1d(n)``: the explicit table of basis functions sampled on pixels, built
  pixel by pixel from SPEC.md S:45/S:78 (2D wavelet = +-2**l on its square; H + left, V + top,
  D + main diagonal) and the 1D analogue (+-2**(l/2), + left).  Rows are in HAAR1 order.
* ``overlap_shift_matrix_*``: the exact coefficient-domain shift operator
  M[i][j] = <psi_i, T_s psi_j> with ``fractions.Fraction`` arithmetic, where T_s translates the
  piecewise-constant function by s pixels (periodic) -- the box projection of DESIGN.md R4 written
  as an integral of overlaps, not as a 2-tap formula.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def _haar1_index_2d(l: int, t: int, i: int, j: int) -> int:
    return 4 ** l * (1 + t) + i * 2 ** l + j


def basis2d(n: int) -> np.ndarray:
    """Psi [N*N][N*N]: row k = basis function k sampled at pixel (r, c) -> column r*N + c."""
    N = 1 << n
    P = np.zeros((N * N, N * N), dtype=np.float64)
    P[0, :] = 1.0
    for l in range(n):
        W = N >> l                      # pixels per square side
        h = W // 2
        for i in range(1 << l):
            for j in range(1 << l):
                for r in range(i * W, (i + 1) * W):
                    for c in range(j * W, (j + 1) * W):
                        top = (r - i * W) < h
                        left = (c - j * W) < h
                        vals = (
                            1.0 if left else -1.0,                    # H: + on left half
                            1.0 if top else -1.0,                     # V: + on top half
                            1.0 if (top == left) else -1.0,           # D: + main diagonal
                        )
                        for t in range(3):
                            P[_haar1_index_2d(l, t, i, j), r * N + c] = vals[t] * 2.0 ** l
    return P


def basis1d(n: int) -> np.ndarray:
    N = 1 << n
    P = np.zeros((N, N), dtype=np.float64)
    P[0, :] = 1.0
    for l in range(n):
        W = N >> l
        for k in range(1 << l):
            for x in range(k * W, (k + 1) * W):
                P[(1 << l) + k, x] = (1.0 if (x - k * W) < W // 2 else -1.0) * 2.0 ** (l / 2.0)
    return P


def basis_int_2d(n: int):
    """Same table with exact integer/Fraction entries (2D values are +-2**l: integers)."""
    return [[Fraction(int(v)) for v in row] for row in basis2d(n)]


def _overlap(p: int, pp: int, s: Fraction, N: int) -> Fraction:
    """Length of [p, p+1) intersect [pp + s, pp + s + 1) on the circle of circumference N."""
    d = (Fraction(p) - pp - s) % N                     # in [0, N)
    ov = Fraction(0)
    if d < 1:
        ov += 1 - d
    if d > N - 1:
        ov += d - (N - 1)
    return ov


def overlap_shift_matrix_1d(n: int, s: Fraction) -> list:
    """M[i][j] = (1/N) sum_p sum_p' psi_i[p] psi_j[p'] |pixel p  cap  (pixel p' + s)|, exact.

    1D basis values are +-2**(l/2); products psi_i psi_j are rational only up to a factor
    2**((l_i + l_j)/2).  We return M in the basis scaled to integers (psi~ = 2**(-l/2) psi, i.e.
    integer +-1 values) together with the scale vector, so the caller composes exactly."""
    N = 1 << n
    tab = np.sign(basis1d(n)).astype(int)              # +-1 / 0 pattern, scaling row 1
    ov = [[_overlap(p, pp, s, N) for pp in range(N)] for p in range(N)]
    M = [[Fraction(0)] * N for _ in range(N)]
    for i in range(N):
        for j in range(N):
            acc = Fraction(0)
            for p in range(N):
                if tab[i][p] == 0:
                    continue
                for pp in range(N):
                    if tab[j][pp] == 0 or ov[p][pp] == 0:
                        continue
                    acc += tab[i][p] * tab[j][pp] * ov[p][pp]
            M[i][j] = acc / N
    return M


def level_1d(k: int) -> int:
    return 0 if k == 0 else k.bit_length() - 1


def exact_shift_operator_1d(n: int, s: Fraction) -> np.ndarray:
    """S[i][j] = <psi_i, T_s psi_j> in the unit-interval basis, from the exact overlap matrix of
    the integer-valued pattern basis psi~ (psi_k = 2**(l_k/2) psi~_k):
    S[i][j] = 2**((l_i + l_j)/2) * M~[i][j]."""
    N = 1 << n
    M = overlap_shift_matrix_1d(n, s)
    S = np.zeros((N, N))
    for i in range(N):
        for j in range(N):
            S[i, j] = float(M[i][j]) * 2.0 ** ((level_1d(i) + level_1d(j)) / 2.0)
    return S


def overlap_shift_matrix_2d(n: int, sy: Fraction, sx: Fraction) -> list:
    """M[i][j] = (1/N**2) sum_{pixels} psi_i psi_j' overlap, exact Fractions (2D values are
    integers +-2**l, so everything is rational)."""
    N = 1 << n
    B = basis2d(n).astype(np.int64)
    K = N * N
    ovr = [[_overlap(p, pp, sy, N) for pp in range(N)] for p in range(N)]
    ovc = [[_overlap(p, pp, sx, N) for pp in range(N)] for p in range(N)]
    # translated basis function j evaluated as an integral over destination pixel (r, c):
    # (T_s psi_j)[r, c] = sum_{r', c'} psi_j[r', c'] ovr[r][r'] ovc[c][c']
    M = [[Fraction(0)] * K for _ in range(K)]
    for j in range(K):
        pj = B[j].reshape(N, N)
        moved = [[Fraction(0)] * N for _ in range(N)]
        for r in range(N):
            for c in range(N):
                acc = Fraction(0)
                for rr in range(N):
                    if ovr[r][rr] == 0:
                        continue
                    for cc in range(N):
                        if ovc[c][cc] == 0 or pj[rr, cc] == 0:
                            continue
                        acc += int(pj[rr, cc]) * ovr[r][rr] * ovc[c][cc]
                moved[r][c] = acc
        for i in range(K):
            pi = B[i].reshape(N, N)
            acc = Fraction(0)
            for r in range(N):
                for c in range(N):
                    if pi[r, c] != 0 and moved[r][c] != 0:
                        acc += int(pi[r, c]) * moved[r][c]
            M[i][j] = acc / (N * N)
    return M


def apply_fraction_matrix(M: list, c: list) -> list:
    return [sum((M[i][j] * c[j] for j in range(len(c))), Fraction(0)) for i in range(len(M))]
