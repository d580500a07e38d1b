"""Pins of the rotation oracle and of the smooth-map generator, -m "not gpu".

* rotated angles: SPEC.md S:185 (alpha = 20 deg at (pi/2, 0) -> (pi/2 + 20 deg, 0)), identity,
  the inverse rotation, orthogonality of R_x (great-circle distances preserved);
* elevate_pixels: identity is an exact copy, constants stay constant, alpha = pi maps the map to
  itself upside down with phi mirrored through pi (closed form);
* rotate_coeffs: alpha = 0 with an integer azimuth shift is the exact circular column shift of the
  pixel map, and alpha = 0, beta = 0 is the identity on coefficients;
* synth.smooth_sphere_maps equals the forward transform of its closed-form cell means;
* the chain-rule algorithm (rotate_coeffs_chain): exact cases (identity, constants, integer
  azimuths, the half turn), convergence to the analytic rotation, and each stage on its own --
  the recursion against forward2d on exact fields, the periodic closure (identity on exact fields,
  a strict improvement toward the analytic rotation, applied inside the chain), the dead last
  row of Y, and the DC rule's level cap (reads exactly the levels below min(n, 6)).
"""
import math

import numpy as np

import synth
from oracle import haar, rotate


def test_rotated_angles_examples():
    a = math.radians(20.0)
    Th, Ph = rotate.rotated_angles(math.pi / 2, 0.0, a)
    assert abs(Th - (math.pi / 2 + a)) < 1e-12 and abs(Ph) < 1e-12
    th = np.linspace(0.1, 3.0, 7)
    ph = np.linspace(0.2, 6.0, 7)
    T0, P0 = rotate.rotated_angles(th, ph, 0.0)
    np.testing.assert_allclose(T0, th, atol=1e-12)
    np.testing.assert_allclose(P0, ph, atol=1e-12)
    T1, P1 = rotate.rotated_angles(th, ph, 0.7)
    T2, P2 = rotate.rotated_angles(T1, P1, -0.7)
    np.testing.assert_allclose(T2, th, atol=1e-10)
    np.testing.assert_allclose(np.mod(P2 - ph + np.pi, 2 * np.pi) - np.pi, 0.0, atol=1e-10)


def _dir(t, p):
    return np.stack([np.sin(t) * np.sin(p), np.cos(t), np.sin(t) * np.cos(p)], axis=-1)


def test_rotation_preserves_angles_between_points():
    rng = np.random.default_rng(0)
    t = rng.uniform(0.05, 3.0, (2, 50))
    p = rng.uniform(0.0, 6.2, (2, 50))
    T, P = rotate.rotated_angles(t, p, -1.1)
    before = np.sum(_dir(t[0], p[0]) * _dir(t[1], p[1]), axis=-1)
    after = np.sum(_dir(T[0], P[0]) * _dir(T[1], P[1]), axis=-1)
    np.testing.assert_allclose(after, before, atol=1e-12)


def test_elevate_identity_constant_and_half_turn():
    rng = np.random.default_rng(1)
    N = 16
    f = rng.normal(size=(N, N))
    np.testing.assert_allclose(rotate.elevate_pixels(f, 0.0), f, atol=1e-12)
    np.testing.assert_allclose(rotate.elevate_pixels(np.full((N, N), 2.5), 0.9), 2.5, atol=1e-12)
    # alpha = pi: (theta, phi) -> (pi - theta, pi - phi): row r -> N-1-r, column c -> N/2-1-c (mod N)
    g = rotate.elevate_pixels(f, math.pi)
    want = f[::-1][:, (N // 2 - 1 - np.arange(N)) % N]
    np.testing.assert_allclose(g, want, atol=1e-9)


def test_rotate_coeffs_identity_and_integer_azimuth():
    c = synth.smooth_sphere_maps(7, 1, 4)[0].astype(np.float64)
    np.testing.assert_allclose(rotate.rotate_coeffs(c, 0.0, 0.0), c, atol=1e-12)
    N = 16
    pix = haar.inverse2d(c)
    got = haar.inverse2d(rotate.rotate_coeffs(c, 0.0, 3 * 2 * math.pi / N))
    np.testing.assert_allclose(got, np.roll(pix, 3, axis=1), atol=1e-12)      # f'(x) = f(x - 3)


def test_psnr_definition():
    c = synth.smooth_sphere_maps(8, 1, 3)[0].astype(np.float64)
    assert rotate.psnr(c, c) == float("inf")
    d = c.copy()
    d[0] += 0.01                                       # every pixel moves by 0.01
    peak = np.abs(haar.inverse2d(c)).max()
    assert abs(rotate.psnr(d, c) - 10 * np.log10(peak ** 2 / 1e-4)) < 1e-9


def test_smooth_maps_are_cell_integrals():
    for n in (3, 5):
        c = synth.smooth_sphere_maps(3, 2, n)
        m = synth.smooth_sphere_cell_means(3, 2, n)
        for k in range(2):
            np.testing.assert_allclose(haar.forward2d(m[k]), c[k], atol=3e-7)


def test_smooth_eval_matches_cell_means():
    """the point evaluator integrates (Gauss-Legendre, 4 x 4 per cell) to the closed-form cell means"""
    n, N = 4, 16
    g, w = np.polynomial.legendre.leggauss(4)
    th = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * np.pi / N        # [N][4]
    ph = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * 2 * np.pi / N
    vals = synth.smooth_sphere_eval(5, 1, th[:, None, :, None], ph[None, :, None, :])
    means = np.einsum("rcab,a,b->rc", vals, w, w) / 4.0
    np.testing.assert_allclose(means, synth.smooth_sphere_cell_means(5, 2, n)[1], atol=1e-9)


# ------------------------------------------------------------- the paper's algorithm (chain rule)

def test_chain_identity_constant_and_azimuth():
    c = synth.smooth_sphere_maps(21, 1, 4)[0].astype(np.float64)
    np.testing.assert_allclose(rotate.rotate_coeffs_chain(c, 0.0, 0.0), c, atol=1e-12)
    N = 16
    const = haar.forward2d(np.full((N, N), -1.75))
    np.testing.assert_allclose(rotate.rotate_coeffs_chain(const, 0.83, -2.1), const, atol=1e-12)
    pix = haar.inverse2d(c)
    got = haar.inverse2d(rotate.rotate_coeffs_chain(c, 0.0, -5 * 2 * math.pi / N))
    np.testing.assert_allclose(got, np.roll(pix, -5, axis=1), atol=1e-12)


def test_chain_half_turn_is_the_exact_flip():
    """alpha = pi maps every sample of the chain rule onto the grid: (theta, phi) -> (pi - theta,
    pi - phi), row r -> N-1-r, column c -> N/2-1-c; the result is that pixel permutation exactly
    (white noise, so every field value is exercised)"""
    rng = np.random.default_rng(22)
    for N in (8, 32):
        f = rng.normal(size=(N, N))
        got = haar.inverse2d(rotate.rotate_coeffs_chain(haar.forward2d(f), math.pi, 0.0))
        want = f[::-1][:, (N // 2 - 1 - np.arange(N)) % N]
        np.testing.assert_allclose(got, want, atol=1e-10)


def _analytic_truth(seed, k, n, alpha, beta):
    """cell means of the exactly rotated analytic map (Gauss-Legendre 4 x 4 per pixel)"""
    N = 1 << n
    g, w = np.polynomial.legendre.leggauss(4)
    th = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * np.pi / N
    ph = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * 2 * np.pi / N - beta
    T, P = np.broadcast_arrays(th[:, None, :, None], ph[None, :, None, :])
    Th, Ph = rotate.rotated_angles(T, P, alpha)
    vals = synth.smooth_sphere_eval(seed, k, Th, Ph)
    return np.einsum("rcab,a,b->rc", vals, w, w) / 4.0


def test_chain_converges_to_the_analytic_rotation():
    """first order in the pixel size (R25): against the analytic rotation of smooth maps
    the PSNR rises with N (measured medians 31.8 / 38.5 / 43.9 dB at N = 16 / 32 / 64; the
    floors catch a dropped term, a sign or a transposed field, which stall or collapse it)"""
    med = []
    for n in (4, 5, 6):
        ang = synth.rotation_angles(23, 4)
        c = synth.smooth_sphere_maps(24, 4, n)
        ps = []
        for b in range(4):
            got = haar.inverse2d(rotate.rotate_coeffs_chain(c[b], *ang[b]))
            truth = _analytic_truth(24, b, n, *ang[b])
            ps.append(10 * np.log10(np.abs(truth).max() ** 2 / np.mean((got - truth) ** 2)))
        med.append(float(np.median(ps)))
    print(med)
    assert med[0] < med[1] < med[2]
    assert med[0] >= 28.0 and med[1] >= 34.0 and med[2] >= 40.0


# ------------------------------------------- the chain-rule stages pinned one by one

def _exact_fields(g):
    """periodic difference fields of a pixel map: X = g - g(c+1), Y = g - g(r+1)"""
    return g - np.roll(g, -1, axis=1), g - np.roll(g, -1, axis=0)


def test_bottom_up_of_exact_fields_is_the_forward_transform():
    """step 5 alone: on the exact periodic fields of any map the [1,1] x [1,2,1] recursion returns
    that map's Haar details -- pinned against forward2d (itself pinned by the basis brute force) --
    and the level-0 residuals vanish"""
    rng = np.random.default_rng(31)
    for n in (1, 2, 3, 5, 7):
        g = rng.normal(size=(1 << n, 1 << n))
        details, res = rotate.fields_bottom_up(*_exact_fields(g))
        got = haar.pack2d(float(g.mean()), details)
        np.testing.assert_allclose(got, haar.forward2d(g), atol=1e-12)
        np.testing.assert_allclose(res, 0.0, atol=1e-9)


def test_last_row_of_y_never_reaches_an_output():
    """why Y_g needs no closure (R27): its last row enters only the odd rows of every
    coarser Y, which no V detail reads -- any value there changes the level-0 residual alone"""
    rng = np.random.default_rng(32)
    for n in (3, 6):
        X, Y = _exact_fields(rng.normal(size=(1 << n, 1 << n)))
        d0, r0 = rotate.fields_bottom_up(X, Y)
        Y2 = Y.copy()
        Y2[-1] = rng.normal(size=1 << n) * 100.0
        d1, r1 = rotate.fields_bottom_up(X, Y2)
        for a, b in zip(d0, d1):
            for u, v in zip(a, b):
                np.testing.assert_array_equal(u, v)
        assert abs(r1[1] - r0[1]) > 1.0


def test_closure_is_the_identity_on_exact_fields_and_zeroes_row_sums():
    """step 3: the exact X field of a periodic map already sums to 0 along each row (a telescoping
    sum), so the closure leaves it unchanged (a closure on the wrong axis, a wrong sign or scale
    would not); on the chain rule's raw field it removes nonzero row sums"""
    rng = np.random.default_rng(33)
    g = rng.normal(size=(32, 32))
    X, _ = _exact_fields(g)
    np.testing.assert_allclose(rotate.periodic_closure(X), X, atol=1e-13)
    f = haar.inverse2d(synth.smooth_sphere_maps(34, 1, 5)[0].astype(np.float64))
    Xr, _ = rotate.chain_rule_fields(f, 0.9)
    assert np.abs(Xr.sum(axis=1)).max() > 1e-4
    np.testing.assert_allclose(rotate.periodic_closure(Xr).sum(axis=1), 0.0, atol=1e-12)


def _analytic_point_fields(seed, k, n, alpha):
    """exact X field of the rotated analytic map sampled at pixel centres"""
    N = 1 << n
    th = (np.arange(N) + 0.5) * np.pi / N
    ph = (np.arange(N) + 0.5) * 2 * np.pi / N
    T, P = np.meshgrid(th, ph, indexing="ij")
    Th, Ph = rotate.rotated_angles(T, P, alpha)
    g = synth.smooth_sphere_eval(seed, k, Th, Ph)
    return g - np.roll(g, -1, axis=1)


def test_closure_moves_chain_fields_toward_the_exact_rotation():
    """the reason for R27: the exact rotated field has zero row sums, so projecting the chain
    rule's raw field onto zero-row-sum fields strictly reduces its distance to the truth (the
    analytic map rotated exactly, sampled at the pixel centres) -- the raw row sums are pure error"""
    for n in (5, 6):
        c = synth.smooth_sphere_maps(35, 3, n)
        ang = synth.rotation_angles(36, 3)
        for b in range(3):
            f = haar.inverse2d(c[b].astype(np.float64))
            Xr, _ = rotate.chain_rule_fields(f, ang[b][0])
            Xt = _analytic_point_fields(35, b, n, ang[b][0])
            e_raw = np.linalg.norm(Xr - Xt)
            e_closed = np.linalg.norm(rotate.periodic_closure(Xr) - Xt)
            assert e_closed < e_raw * (1 - 1e-6), (n, b, e_raw, e_closed)


def test_chain_is_the_composition_of_its_stages():
    """rotate_coeffs_chain applies every stage (a dropped closure or a different DC rule fails
    here): the composition written out from the pinned stages, and the same without the closure
    differs"""
    c = synth.smooth_sphere_maps(37, 2, 5)
    ang = synth.rotation_angles(38, 2)
    for b in range(2):
        f = haar.inverse2d(c[b].astype(np.float64))
        Xr, Yr = rotate.chain_rule_fields(f, ang[b][0])
        N = f.shape[0]
        sh = ang[b][1] * N / (2 * np.pi)
        d, _ = rotate.fields_bottom_up(rotate.periodic_closure(Xr), Yr)
        want = shift_coeffs2d(haar.pack2d(rotate.rotated_dc(f, ang[b][0]), d), 0.0, sh)
        got = rotate.rotate_coeffs_chain(c[b], *ang[b])
        np.testing.assert_allclose(got, want, atol=1e-12)
        d_open, _ = rotate.fields_bottom_up(Xr, Yr)
        unclosed = shift_coeffs2d(haar.pack2d(rotate.rotated_dc(f, ang[b][0]), d_open), 0.0, sh)
        assert np.abs(unclosed - got).max() > 1e-6


def shift_coeffs2d(c, sy, sx):
    from oracle import shift
    return shift.shift_coeffs2d(c, sy, sx)


def _perturbed_dc(c, level, alpha, rng):
    """rotated_dc of the map before and after a random change of one detail coefficient at `level`"""
    n = haar.log2_exact(int(round(np.sqrt(c.size))))
    idx = 4 ** level * (1 + rng.integers(0, 3)) + rng.integers(0, 4 ** level)
    d = c.astype(np.float64).copy()
    d[idx] += 0.5
    return (rotate.rotated_dc(haar.inverse2d(c.astype(np.float64)), alpha),
            rotate.rotated_dc(haar.inverse2d(d), alpha))


def test_dc_reads_exactly_the_levels_below_six():
    """R27 / S:301: the scaling coefficient is the mean of the level-min(n, 6) approximation
    resampled at the rotated pixel centres.  So at n = 7 and 8 (where the cap binds) no detail at
    level >= 6 can move it, while every coarser level does (a rule reading level 5 or level n
    fails one of the two); at n = 5 every level moves it"""
    rng = np.random.default_rng(39)
    for n in (7, 8):
        c = synth.smooth_sphere_maps(40, 1, n)[0]
        for level in (6, n - 1):
            a, b = _perturbed_dc(c, level, 0.7, rng)
            assert abs(a - b) <= 1e-13 * abs(a), (n, level)
        for level in (5, 3):
            a, b = _perturbed_dc(c, level, 0.7, rng)
            assert abs(a - b) > 1e-7, (n, level, a, b)
    c = synth.smooth_sphere_maps(41, 1, 5)[0]
    for level in (4, 2):
        a, b = _perturbed_dc(c, level, 0.7, rng)
        assert abs(a - b) > 1e-7


def test_dc_exact_cases():
    """alpha = 0 samples every cell at its centre: the DC is the map's mean exactly, at every n
    (including n > 6, where the level-6 cell means average to the same mean); a constant stays"""
    for n in (3, 6, 8):
        c = synth.smooth_sphere_maps(42, 1, n)[0].astype(np.float64)
        f = haar.inverse2d(c)
        assert abs(rotate.rotated_dc(f, 0.0) - c[0]) < 1e-12
        assert abs(rotate.rotated_dc(np.full_like(f, 3.25), 1.234) - 3.25) < 1e-12


def test_chain_output_dc_ignores_fine_levels():
    """end to end at n = 8: changing level-6 and level-7 details of the input leaves the output's
    scaling coefficient unchanged"""
    rng = np.random.default_rng(43)
    c = synth.smooth_sphere_maps(44, 1, 8)[0].astype(np.float64)
    d = c.copy()
    d[4 ** 6:] += rng.normal(size=c.size - 4 ** 6) * 0.01
    a = rotate.rotate_coeffs_chain(c, 0.6, 1.0)[0]
    b = rotate.rotate_coeffs_chain(d, 0.6, 1.0)[0]
    assert abs(a - b) <= 1e-13 * abs(a)          # fp64 rounding of the cell means only
