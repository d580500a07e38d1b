"""Pins of the oracle's relight (-m "not gpu"): the double product equals the pixel-domain
integral of the two functions (orthonormality, built from the brute basis table), DC invariance
under any shift, unit vectors pick coefficients, integer shifts preserve <L, T> when both move,
bilinearity, and the fused per-vertex form against an explicit per-vertex loop."""
import numpy as np
import pytest

import brute
import synth
from oracle import haar, relight, shift


def test_double_product_is_pixel_integral():
    """sum_k L_k T_k = mean over pixels of f_L f_T (Parseval form, basis table from brute)."""
    n, N = 3, 8
    P = brute.basis2d(n)
    rng = np.random.default_rng(1)
    L = rng.normal(size=(1, 1, N * N))
    T = rng.normal(size=(5, N * N))
    R = relight.relight(T, L, 1, N * N)
    fL = P.T @ L[0, 0]
    for v in range(5):
        fT = P.T @ T[v]
        assert abs(R[v, 0] - np.mean(fL * fT)) < 1e-12


def test_unit_vectors_and_dc_invariance():
    rng = np.random.default_rng(2)
    L = rng.normal(size=(3, 2, 64))
    e0 = np.zeros((1, 128)); e0[0, 0] = 1.0
    ek = np.zeros((1, 128)); ek[0, 64 + 37] = 1.0
    np.testing.assert_allclose(relight.relight(e0, L, 2, 64)[0], L[:, 0, 0])
    np.testing.assert_allclose(relight.relight(ek, L, 2, 64)[0], L[:, 1, 37])
    for s in [(0.3, 4.7), (-2.0, 1.0), (5.5, 5.5)]:
        Ls = shift.shift_coeffs2d(L[0, 0], *s)
        assert abs(Ls[0] - L[0, 0, 0]) < 1e-13                  # r(e0) = scaling for any shift


def test_integer_shift_preserves_inner_product():
    rng = np.random.default_rng(3)
    L, T = rng.normal(size=(2, 256))
    for s in [(3.0, -7.0), (8.0, 1.0)]:
        lhs = np.dot(shift.shift_coeffs2d(L, *s), shift.shift_coeffs2d(T, *s))
        assert abs(lhs - np.dot(L, T)) < 1e-11


def test_band_prefix_and_bilinearity():
    rng = np.random.default_rng(4)
    L = rng.normal(size=(2, 6, 256))
    T = rng.normal(size=(7, 6 * 16))
    R = relight.relight(T, L, 6, 16)
    manual = np.array([[sum(np.dot(T[v, f * 16:(f + 1) * 16], L[b, f, :16]) for f in range(6))
                        for b in range(2)] for v in range(7)])
    np.testing.assert_allclose(R, manual, atol=1e-12)
    np.testing.assert_allclose(relight.relight(2 * T, L, 6, 16), 2 * R)
    np.testing.assert_allclose(relight.relight(T, -3 * L, 6, 16), -3 * R)


def test_relight_shifted_matches_loop():
    n, N, F = 3, 8, 2
    rng = np.random.default_rng(5)
    L = rng.normal(size=(F, N * N))
    T = rng.normal(size=(4, F * N * N))
    sv = np.array([[0.0, 0.0], [1.5, -2.25], [8.0, 3.0], [0.125, 7.5]])
    got = relight.relight_shifted(T, L, sv)
    for v in range(4):
        Lp = np.concatenate([shift.shift_coeffs2d(L[f], *sv[v]) for f in range(F)])
        assert abs(got[v] - np.dot(Lp, T[v])) < 1e-12
    # zero shift: plain dot
    np.testing.assert_allclose(relight.relight_shifted(T, L, np.zeros((4, 2))), T @ L.reshape(-1), atol=1e-12)


def test_sparse_relight_equals_dense_scatter():
    """The sparse double product equals the dense one with the (idx, val) pairs scattered into a
    dense transfer row (duplicates add), computed with BLAS."""
    n, F, B = 4, 6, 3
    idx, val = synth.sparse_transfer_rows(9, 0, 50, F, n, 120)
    L = synth.light_pyramids(10, B, F, n).reshape(B, -1)
    dense = np.zeros((50, F * 4 ** n))
    for v in range(50):
        np.add.at(dense[v], idx[v].astype(np.int64), val[v].astype(np.float64))
    np.testing.assert_allclose(relight.relight_sparse(idx, val, L), dense @ L.T.astype(np.float64), rtol=1e-12,
                               atol=1e-12)


def test_sparse_generator_structure():
    n, F, K = 5, 6, 200
    idx, val = synth.sparse_transfer_rows(11, 3, 20, F, n, K, dense_levels=2)
    assert idx.dtype == np.int32 and val.dtype == np.float32
    assert idx.min() >= 0 and idx.max() < F * 4 ** n
    dense_part = idx[:, :F * 16]
    np.testing.assert_array_equal(dense_part, np.broadcast_to(
        (np.arange(F)[:, None] * 4 ** n + np.arange(16)[None, :]).reshape(-1), dense_part.shape))
    coef = idx % 4 ** n
    lev = synth.level_of_index_2d(coef)
    assert np.all(np.abs(val) <= 2.0 ** -lev)
    assert np.all(val[coef == 0] >= 0)
    np.testing.assert_array_equal(synth.sparse_transfer_rows(11, 5, 4, F, n, K)[0], idx[2:6])


def test_synth_transfer_is_counter_based_and_exact():
    """Generator determinism: row subsets equal slices of the full matrix; values exact fp32."""
    full = synth.transfer_rows(123, 0, 20, 6, 16)
    sub = synth.transfer_rows(123, 7, 5, 6, 16)
    np.testing.assert_array_equal(full[7:12], sub)
    assert np.all(full[:, ::16] >= 0)                               # scaling entries |u|
    lev = synth.level_of_index_2d(np.arange(16))
    assert np.all(np.abs(full[:, :16]) <= 2.0 ** -lev + 0)
    assert full.dtype == np.float32
