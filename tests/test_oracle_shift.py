"""Pins of the oracle's shift (-m "not gpu"): exact Fraction overlap-integral operators (an
independent brute force of the box projection), SURVEY App. B worked examples, and closed forms
(identity at 0 and N, integer composition, fractional composition closed form, DC invariance,
Parseval for integer shifts, linearity in the fractional part, adjoint, dyadic permutation)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import brute
from oracle import haar, shift

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _op1d(n, s):
    N = 1 << n
    return np.stack([shift.shift_coeffs1d(e, s) for e in np.eye(N)], axis=1)


def _op2d(n, sy, sx):
    N = 1 << n
    return np.stack([shift.shift_coeffs2d(e, sy, sx) for e in np.eye(N * N)], axis=1)


# ----------------------------------------------------------------- exact brute force (T0)

@pytest.mark.parametrize("s", ["0", "1", "3", "1/2", "5/4", "7/3", "-9/4", "8", "17/2", "-1"])
def test_1d_n8_operator_equals_fraction_overlaps(s):
    """Whole 8x8 operator, every basis vector: oracle == <psi_i, T_s psi_j> (exact overlaps)."""
    S = brute.exact_shift_operator_1d(3, Fraction(s))
    np.testing.assert_allclose(_op1d(3, float(Fraction(s))), S, atol=2e-15)


@pytest.mark.parametrize("sy,sx", [("0", "0"), ("1", "0"), ("0", "3"), ("1/2", "0"),
                                   ("1/4", "7/4"), ("5/2", "-3/2"), ("4", "4"), ("-1/8", "9/8")])
def test_2d_4x4_operator_equals_fraction_overlaps(sy, sx):
    M = brute.overlap_shift_matrix_2d(2, Fraction(sy), Fraction(sx))
    S = np.array([[float(x) for x in row] for row in M])
    np.testing.assert_allclose(_op2d(2, float(Fraction(sy)), float(Fraction(sx))), S, atol=2e-15)


def test_2d_8x8_operator_one_fractional_case():
    M = brute.overlap_shift_matrix_2d(3, Fraction(3, 4), Fraction(-5, 2))
    S = np.array([[float(x) for x in row] for row in M])
    np.testing.assert_allclose(_op2d(3, 0.75, -2.5), S, atol=2e-15)


def test_survey_appendix_b_examples():
    g = json.load(open(os.path.join(GOLD, "survey_appB_shifts.json")))
    f1 = np.array(g["1d"]["signal"], float)
    for case in g["1d"]["cases"]:
        s = float(Fraction(case["s"]))
        c = shift.shift_coeffs1d(haar.forward1d(f1), s)
        sc, dets = haar.unpack1d(c)
        assert sc == float(Fraction(g["1d"]["scaling"]))
        for l, d in enumerate(dets):
            np.testing.assert_allclose(d * 2 ** (l / 2), [float(Fraction(x)) for x in case["d"][l]],
                                       atol=1e-14)
    f2 = np.array(g["2d"]["map"], float)
    for case in g["2d"]["cases"]:
        sy, sx = (float(Fraction(x)) for x in case["s"])
        c = shift.shift_coeffs2d(haar.forward2d(f2), sy, sx)
        sc, dets = haar.unpack2d(c)
        assert abs(sc - float(Fraction(g["2d"]["scaling"]))) < 1e-15
        np.testing.assert_allclose([dets[0][t][0, 0] for t in range(3)],
                                   [float(Fraction(x)) for x in case["L0"]], atol=1e-15)
        for t, key in enumerate(["L1H", "L1V", "L1D"]):
            np.testing.assert_allclose(dets[1][t], [[float(Fraction(x)) for x in r] for r in case[key]],
                                       atol=1e-15)
    # the fixture itself agrees with the independent Fraction brute force
    M = brute.overlap_shift_matrix_2d(2, Fraction(1, 2), Fraction(1, 2))
    P = brute.basis2d(2)
    c0 = [Fraction(x).limit_denominator(1 << 20) for x in P @ f2.ravel() / 16]
    c1 = brute.apply_fraction_matrix(M, c0)
    case = g["2d"]["cases"][4]
    assert [str(x) for x in c1[1:4]] == case["L0"]


# ----------------------------------------------------------------- closed forms (T1)

@pytest.mark.parametrize("n", [3, 5])
def test_identity_at_zero_and_N(n):
    N = 1 << n
    c = np.random.default_rng(n).normal(size=N * N)
    for s in [(0.0, 0.0), (float(N), 0.0), (0.0, -float(N)), (2.0 * N, 3.0 * N)]:
        np.testing.assert_allclose(shift.shift_coeffs2d(c, *s), c, atol=1e-12)
    c1 = np.random.default_rng(n + 7).normal(size=N)
    for s in [0.0, float(N), -3.0 * N]:
        np.testing.assert_allclose(shift.shift_coeffs1d(c1, s), c1, atol=1e-12)


def test_integer_composition_and_fraction_with_integer():
    """S_a S_b = S_{a+b} when a or b is an integer."""
    rng = np.random.default_rng(5)
    c = rng.normal(size=256)
    for a, b in [((3.0, -5.0), (7.0, 2.0)), ((0.25, 1.0), (1.0, 6.0)), ((-2.0, 0.0), (0.5, 0.75))]:
        lhs = shift.shift_coeffs2d(shift.shift_coeffs2d(c, *a), *b)
        rhs = shift.shift_coeffs2d(c, a[0] + b[0], a[1] + b[1])
        np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_fractional_composition_closed_form():
    """S_p1 S_p2 = (1-p1)(1-p2) I + [(1-p1)p2 + p1(1-p2)] S_1 + p1 p2 S_2 (1D, per axis)."""
    c = np.random.default_rng(6).normal(size=16)
    for p1, p2 in [(0.3, 0.6), (0.5, 0.5), (0.125, 0.75)]:
        lhs = shift.shift_coeffs1d(shift.shift_coeffs1d(c, p1), p2)
        rhs = ((1 - p1) * (1 - p2) * c + ((1 - p1) * p2 + p1 * (1 - p2)) * shift.shift_coeffs1d(c, 1.0)
               + p1 * p2 * shift.shift_coeffs1d(c, 2.0))
        np.testing.assert_allclose(lhs, rhs, atol=1e-13)
    assert not np.allclose(shift.shift_coeffs1d(shift.shift_coeffs1d(c, 0.5), 0.5),
                           shift.shift_coeffs1d(c, 1.0))


def test_dc_invariance_and_energy():
    rng = np.random.default_rng(7)
    c = rng.normal(size=1024)
    for s in [(3.3, -1.6), (0.5, 0.5), (17.0, 4.0)]:
        out = shift.shift_coeffs2d(c, *s)
        assert abs(out[0] - c[0]) < 1e-13                              # R8: mean preserved
        e_in, e_out = np.sum(c ** 2), np.sum(out ** 2)
        if float(s[0]).is_integer() and float(s[1]).is_integer():
            assert abs(e_out - e_in) < 1e-10 * e_in                    # isometry (Parseval)
        else:
            assert e_out <= e_in * (1 + 1e-12)                         # contraction
    white = rng.normal(size=1 << 14)
    r = np.sum(shift.shift_coeffs1d(white, 0.5) ** 2) / np.sum(white ** 2)
    assert 0.4 < r < 0.55                                              # ~0.46


def test_linear_in_fractional_part():
    """S_{q+phi} = (1-phi) S_q + phi S_{q+1} per axis."""
    c = np.random.default_rng(8).normal(size=64)
    for q, phi in [(2, 0.3), (-3, 0.8), (5, 0.5)]:
        lhs = shift.shift_coeffs2d(c, 0.0, q + phi)
        rhs = (1 - phi) * shift.shift_coeffs2d(c, 0.0, q) + phi * shift.shift_coeffs2d(c, 0.0, q + 1)
        np.testing.assert_allclose(lhs, rhs, atol=1e-13)


def test_adjoint():
    """(S_phi)^T = (1 - phi) I + phi S_{-1} (1D, N = 16, matrix form)."""
    n, phi = 4, 0.35
    A = _op1d(n, phi)
    np.testing.assert_allclose(A.T, (1 - phi) * np.eye(16) + phi * _op1d(n, -1.0), atol=1e-14)


def test_dyadic_levels_are_permutations():
    """Levels l with 2**(n-l) | s are exact circular permutations."""
    n, N = 5, 32
    c = np.random.default_rng(9).normal(size=N * N)
    for qy, qx in [(4, 8), (0, 12), (16, 2), (8, 24)]:
        out = shift.shift_coeffs2d(c, qy, qx)
        _, din = haar.unpack2d(c)
        _, dout = haar.unpack2d(out)
        for l in range(n):
            W = N >> l
            if qy % W == 0 and qx % W == 0:
                for t in range(3):
                    np.testing.assert_allclose(dout[l][t], np.roll(din[l][t], (qy // W, qx // W), (0, 1)),
                                               atol=1e-13)


def test_half_width_shift_negates_1d_level0():
    """1D: shift by N/2 swaps the two halves -> the level-0 detail changes sign (App. B)."""
    c = np.random.default_rng(10).normal(size=16)
    out = shift.shift_coeffs1d(c, 8.0)
    assert abs(out[1] + c[1]) < 1e-14


def test_split_shift_reduction():
    assert shift.split_shift(-1.25, 8) == (6, 0.75)
    assert shift.split_shift(8.0, 8) == (0, 0.0)
    q, p = shift.split_shift(1e-300 - 8.0, 8)
    assert 0 <= q < 8 and 0 <= p < 1


def test_batched_and_band():
    rng = np.random.default_rng(11)
    c = rng.normal(size=(2, 3, 64))
    s = rng.uniform(-5, 5, size=(2, 3, 2))
    out = shift.shift_coeffs(c, s, 2)
    np.testing.assert_allclose(out[1, 2], shift.shift_coeffs2d(c[1, 2], *s[1, 2]))
    band = shift.shift_coeffs(c, s, 2, band_levels=2)
    np.testing.assert_array_equal(band, out[:, :, :16])


# ----------------------------------------------------------------- coarse start (f4, R23)

def test_coarse_start_is_exact_for_dyadic_shifts():
    """Shifts that are multiples of 2**(n-L) move the level-L approximation by whole cells, so the
    coarse start reproduces the exact shift's levels < L (SPEC.md S:277 permutation argument)."""
    n, N = 5, 32
    c = np.random.default_rng(20).normal(size=N * N)
    for L in (2, 3, 4):
        step = 2 ** (n - L)
        for q in [(step, 0), (3 * step, 2 * step), (0, 5 * step), (-step, 7 * step)]:
            exact = shift.shift_coeffs2d(c, *q)[: 4 ** L]
            np.testing.assert_allclose(shift.shift_coeffs_coarse2d(c, L, *q), exact, atol=1e-12)


def test_coarse_start_at_full_level_is_the_exact_shift():
    c = np.random.default_rng(21).normal(size=256)
    for s in [(0.3, 7.25), (-3.5, 1.0)]:
        np.testing.assert_allclose(shift.shift_coeffs_coarse2d(c, 4, *s), shift.shift_coeffs2d(c, *s), atol=1e-12)


def test_coarse_start_equals_shift_of_truncated_map_cells():
    """Independent restatement: the level-L cells are the means of 2**k x 2**k pixel blocks; shift
    that block-mean image by s/2**k with the brute-force Fraction operator of tests/brute.py."""
    n, L = 3, 2
    N = 1 << n
    f = np.random.default_rng(22).integers(-5, 6, size=(N, N)).astype(float)
    P = brute.basis2d(n)
    c = P @ f.ravel() / (N * N)
    cells = f.reshape(4, 2, 4, 2).mean(axis=(1, 3))                  # level-2 approximation
    P2 = brute.basis2d(L)
    c2 = [Fraction(x).limit_denominator(1 << 20) for x in P2 @ cells.ravel() / 16]
    M = brute.overlap_shift_matrix_2d(L, Fraction(3, 4), Fraction(-5, 4))   # s / 2 = (0.75, -1.25)
    expect = np.array([float(x) for x in brute.apply_fraction_matrix(M, c2)])
    np.testing.assert_allclose(shift.shift_coeffs_coarse2d(c, L, 1.5, -2.5), expect, atol=1e-13)
