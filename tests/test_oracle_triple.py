"""Pins of the oracle's triple product, -m "not gpu".

The oracle integrates the product of the three reconstructed functions.  It is pinned to:
* the triple sum sum_ijk C_ijk a_i b_j c_k of eq:tripleSum with every C_ijk integrated
  from the explicit basis table of tests/brute.py (n = 1, 2, 3);
* the Tripling Coefficient Theorem itself: the same integrated C_ijk take exactly the
  values the theorem's three cases give and are zero otherwise;
* SPEC.md S:126 (all three maps [[1,2],[3,4]] -> 25), scaling-only inputs (case (a) -> a b c),
  visibility = 1 (the triple product collapses to the double product), symmetry, trilinearity.
"""
import itertools

import numpy as np
import pytest

import brute
from oracle import relight


def _tripling(n):
    P = brute.basis2d(n)
    N2 = P.shape[1]
    return np.einsum("ip,jp,kp->ijk", P, P, P) / N2, P


def _level_type_cell(idx, n):
    """HAAR1 index -> (level, type, i, j), or None for the scaling function."""
    if idx == 0:
        return None
    l = 0
    while 4 ** (l + 1) <= idx:
        l += 1
    t, r = divmod(idx - 4 ** l, 4 ** l)
    return l, t, r // 2 ** l, r % 2 ** l


def _theorem_value(a, b, c, n, P):
    """C_ijk from the theorem's case analysis alone; the sign in case (c) is the value
    of the coarser function on the pair's square, read from its definition."""
    ids = [a, b, c]
    info = [_level_type_cell(x, n) for x in ids]
    if all(x is None for x in info):
        return 1.0                                                           # case (a)
    if all(x is not None for x in info):
        (l0, t0, i0, j0), (l1, t1, i1, j1), (l2, t2, i2, j2) = info
        if (l0, i0, j0) == (l1, i1, j1) == (l2, i2, j2) and len({t0, t1, t2}) == 3:
            return 2.0 ** l0                                                 # case (b)
    for p, q, r in ((0, 1, 2), (0, 2, 1), (1, 2, 0)):
        if ids[p] == ids[q] and info[p] is not None:
            l, t, i, j = info[p]
            if info[r] is None:
                return 1.0                                                   # case (c), scaling
            lr, tr, ir, jr = info[r]
            if lr < l and (i >> (l - lr)) == ir and (j >> (l - lr)) == jr:
                N = 1 << n
                W = N >> l                                                   # pair's square, pixels
                pix = (i * W) * N + j * W                                    # any pixel inside it
                return float(P[ids[r], pix])                                 # +-2**lr
    return 0.0


@pytest.mark.parametrize("n", [1, 2])
def test_tripling_coefficient_theorem(n):
    C, P = _tripling(n)
    K = 4 ** n
    mism = 0
    for a, b, c in itertools.product(range(K), repeat=3):
        if C[a, b, c] != _theorem_value(a, b, c, n, P):
            mism += 1
    assert mism == 0
    vals = set(np.unique(C).tolist())
    assert vals <= {0.0, 1.0} | {s * 2.0 ** l for l in range(n) for s in (1, -1)}


def test_tripling_theorem_sparsity_n3():
    C, P = _tripling(3)
    nz = np.argwhere(C != 0)
    rng = np.random.default_rng(0)
    for a, b, c in nz[rng.choice(len(nz), 400, replace=False)]:
        assert C[a, b, c] == _theorem_value(a, b, c, 3, P)
    for a, b, c in rng.integers(0, 64, size=(3000, 3)):
        assert C[a, b, c] == _theorem_value(a, b, c, 3, P)


@pytest.mark.parametrize("n,faces", [(1, 1), (2, 2), (3, 1)])
def test_oracle_equals_triple_sum(n, faces):
    C, _ = _tripling(n)
    K = 4 ** n
    rng = np.random.default_rng(10 + n)
    V, B = 3, 2
    rho = rng.normal(size=(V, faces * K))
    vis = rng.normal(size=(V, faces * K))
    L = rng.normal(size=(B, faces, K))
    got = relight.relight_triple(rho, vis, L, faces, K)
    for v in range(V):
        for b in range(B):
            want = sum(np.einsum("ijk,i,j,k->", C, L[b, f], rho[v, f * K:(f + 1) * K], vis[v, f * K:(f + 1) * K])
                       for f in range(faces))
            assert abs(got[v, b] - want) < 1e-12 * max(1.0, abs(want))


def test_spec_example_and_scaling_only():
    P = brute.basis2d(1)
    m = np.array([1.0, 2.0, 3.0, 4.0])
    c = P @ m / 4.0                                                          # forward = Psi f / N^2
    got = relight.relight_triple(c[None], c[None], c[None, None], 1, 4)
    assert abs(got[0, 0] - 25.0) < 1e-13
    e = np.zeros((1, 16))
    a, b, cc = e.copy(), e.copy(), e.copy()
    a[0, 0], b[0, 0], cc[0, 0] = 1.5, -2.0, 0.25
    assert relight.relight_triple(a, b, cc[:, None, :], 1, 16)[0, 0] == 1.5 * -2.0 * 0.25


def test_unit_visibility_reduces_to_double_product_and_symmetry():
    rng = np.random.default_rng(3)
    F, K, V, B = 2, 64, 4, 3
    rho = rng.normal(size=(V, F * K))
    L = rng.normal(size=(B, F, K))
    one = np.zeros((V, F * K))
    one[:, ::K] = 1.0
    np.testing.assert_allclose(relight.relight_triple(rho, one, L, F, K), relight.relight(rho, L, F, K),
                               rtol=1e-12, atol=1e-12)
    vis = rng.normal(size=(V, F * K))
    R = relight.relight_triple(rho, vis, L, F, K)
    np.testing.assert_allclose(relight.relight_triple(vis, rho, L, F, K), R, rtol=1e-12, atol=1e-12)
    # swap the light with the BRDF of vertex 0
    R2 = relight.relight_triple(L[0].reshape(1, -1), vis[:1], rho[:1].reshape(1, F, K), F, K)
    assert abs(R2[0, 0] - R[0, 0]) < 1e-11
    np.testing.assert_allclose(relight.relight_triple(2 * rho, vis, -L, F, K), -2 * R, rtol=1e-12, atol=1e-12)
