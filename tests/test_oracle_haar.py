"""Pins of the oracle's Haar transforms (-m "not gpu").  Each pin is independent of the oracle:
SPEC worked examples, the explicit basis table built pixel by pixel (tests/brute.py), closed forms
(constant map, Parseval, orthonormality)."""
import json
import os

import numpy as np
import pytest

import brute
from oracle import haar

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_worked_examples():
    """SPEC.md S:48."""
    g = json.load(open(os.path.join(GOLD, "spec_haar2d_examples.json")))
    for ex in g["forward"]:
        np.testing.assert_array_equal(haar.forward2d(np.array(ex["map"], float)), ex["coeffs"])
    for ex in g["inverse"]:
        np.testing.assert_array_equal(haar.inverse2d(np.array(ex["coeffs"], float)), ex["map"])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_forward2d_equals_basis_table(n):
    """c_k = mean over pixels of f * psi_k with psi from the literal definition."""
    N = 1 << n
    P = brute.basis2d(n)
    rng = np.random.default_rng(n)
    for _ in range(4):
        f = rng.normal(size=(N, N))
        np.testing.assert_allclose(haar.forward2d(f), P @ f.ravel() / (N * N), atol=1e-14)
        c = rng.normal(size=N * N)
        np.testing.assert_allclose(haar.inverse2d(c).ravel(), P.T @ c, atol=1e-13)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_forward1d_equals_basis_table(n):
    N = 1 << n
    P = brute.basis1d(n)
    rng = np.random.default_rng(10 + n)
    for _ in range(4):
        f = rng.normal(size=N)
        np.testing.assert_allclose(haar.forward1d(f), P @ f / N, atol=1e-14)
        c = rng.normal(size=N)
        np.testing.assert_allclose(haar.inverse1d(c), P.T @ c, atol=1e-13)


@pytest.mark.parametrize("n", [2, 3])
def test_basis_orthonormal_unit_square(n):
    """(1/N^2) Psi Psi^T = I: the unit-square basis is orthonormal (SPEC.md S:33 Parseval)."""
    N = 1 << n
    P = brute.basis2d(n)
    np.testing.assert_allclose(P @ P.T / (N * N), np.eye(N * N), atol=1e-14)
    P1 = brute.basis1d(n)
    np.testing.assert_allclose(P1 @ P1.T / N, np.eye(N), atol=1e-14)


@pytest.mark.parametrize("n", [1, 4, 7])
def test_constant_map_pure_scaling(n):
    """constant map -> scaling c, all details 0."""
    N = 1 << n
    c = haar.forward2d(np.full((N, N), 3.75))
    assert c[0] == 3.75 and np.all(c[1:] == 0.0)


@pytest.mark.parametrize("n", [3, 6, 9])
def test_round_trip_and_parseval(n):
    """round trip 1e-12, Parseval (mean square) 1e-9."""
    N = 1 << n
    f = np.random.default_rng(n).normal(size=(N, N)) * 10
    c = haar.forward2d(f)
    assert np.max(np.abs(haar.inverse2d(c) - f)) <= 1e-12 * np.max(np.abs(f))
    assert abs(np.sum(c ** 2) - np.mean(f ** 2)) <= 1e-9 * np.mean(f ** 2)
    f1 = np.random.default_rng(n + 1).normal(size=N * N)
    c1 = haar.forward1d(f1)
    assert np.max(np.abs(haar.inverse1d(c1) - f1)) <= 1e-12 * np.max(np.abs(f1))
    assert abs(np.sum(c1 ** 2) - np.mean(f1 ** 2)) <= 1e-9 * np.mean(f1 ** 2)


def test_linearity():
    """SPEC.md S:73."""
    rng = np.random.default_rng(3)
    a, b = rng.normal(size=(2, 16, 16))
    np.testing.assert_allclose(haar.forward2d(2.5 * a - 0.75 * b),
                               2.5 * haar.forward2d(a) - 0.75 * haar.forward2d(b), atol=1e-12)


def test_haar1_layout_and_level_ranges():
    """HAAR1 order: a single level-l H/V/D coefficient synthesises +-2**l on one square."""
    n, N = 3, 8
    for l in range(n):
        for t in range(3):
            for (i, j) in [(0, 0), ((1 << l) - 1, 0)]:
                c = np.zeros(N * N)
                c[4 ** l * (1 + t) + i * (1 << l) + j] = 1.0
                f = haar.inverse2d(c)
                W = N >> l
                sq = f[i * W:(i + 1) * W, j * W:(j + 1) * W]
                assert np.all(np.abs(sq) == 2.0 ** l)
                assert np.count_nonzero(f) == W * W
                h = W // 2
                q = (sq[0, 0], sq[0, h], sq[h, 0], sq[h, h])           # TL, TR, BL, BR
                expect = [(1, -1, 1, -1), (1, 1, -1, -1), (1, -1, -1, 1)][t]
                assert tuple(np.sign(q)) == expect


def test_non_power_of_two_rejected():
    with pytest.raises(ValueError):
        haar.forward2d(np.zeros((6, 6)))
    with pytest.raises(ValueError):
        haar.forward1d(np.zeros(12))
