"""GPU parity of haar_shift_coeffs (the CUDA path through the C ABI) against the fp64 oracle on the
same seeded fp32 inputs (-m gpu).  Gate (BASELINE.json north_star): relative L2 error <= 1e-5 per
output tensor; here checked per (frame, face) pyramid, which is stricter."""
import numpy as np
import pytest

import synth
from oracle import shift as oshift

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _hs():
    import paper_1705_07272_b200 as hs
    return hs


def _run(coeffs, shifts, ndim, band=None):
    import torch
    out = _hs().haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float32)).cuda(),
                                  shifts, ndim, band)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _rel(got, ref, axis=-1):
    num = np.linalg.norm(got - ref, axis=axis)
    den = np.linalg.norm(ref, axis=axis)
    return num / np.maximum(den, 1e-300)


def _signals(n, ndim, seed):
    K = (4 if ndim == 2 else 2) ** n
    norm = synth.random_signals(seed, 8, K, "normal")
    ints = synth.random_signals(seed + 1, 8, K, "int")
    basis = np.eye(K, dtype=np.float32)[: min(K, 16)]
    return np.concatenate([norm, ints, basis])


def test_c1_1d_all_shifts_n8():
    sig = _signals(3, 1, 11)
    shifts = synth.c1_shifts_1d()
    B, F = len(shifts), len(sig)
    coeffs = np.broadcast_to(sig[None], (B, F, 8))
    sh = np.broadcast_to(shifts[:, None, None], (B, F, 1))
    got = _run(coeffs, sh, 1)
    ref = oshift.shift_coeffs(coeffs, sh, 1)
    assert _rel(got, ref).max() <= TOL


def test_c1_2d_all_shifts_4x4():
    sig = _signals(2, 2, 12)
    shifts = synth.c1_shifts_2d()
    B, F = len(shifts), len(sig)
    coeffs = np.broadcast_to(sig[None], (B, F, 16))
    sh = np.broadcast_to(shifts[:, None, :], (B, F, 2))
    got = _run(coeffs, sh, 2)
    ref = oshift.shift_coeffs(coeffs, sh, 2)
    assert _rel(got, ref).max() <= TOL


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_2d_every_size_mixed_shifts(n):
    """White-noise pyramids at every size N = 2 .. 512 (the fields are fp64 at every size, so the
    N = 512 case no longer needs the HDR-shaped light a round-1 fp32 build fell back to); HDR-
    shaped light at N = 512 as well."""
    N = 1 << n
    rng = np.random.default_rng(100 + n)
    shifts = [(0, 0), (N, -N), (1, 0), (0, 1), (N // 2, 0), (0, N // 4 if N >= 4 else 1), (3.3, -1.6),
              (0.5, 0.5), (N - 0.25, 0.125), (-7.75, 2 * N + 0.5)]
    shifts += [tuple(x) for x in rng.uniform(-2 * N, 2 * N, size=(6, 2))]
    shifts += [tuple(x) for x in rng.integers(-N, 2 * N, size=(4, 2)).astype(float)]
    B, F = len(shifts), 2
    coeffs = synth.random_signals(200 + n, B * F, N * N).reshape(B, F, N * N)
    if n >= 9:   # both kinds at the largest size of this sweep
        coeffs = np.concatenate([coeffs, synth.light_pyramids(200 + n, B, F, n)], axis=1)
        F = 2 * F
    sh = np.broadcast_to(np.array(shifts, dtype=np.float64)[:, None, :], (B, F, 2)).copy()
    got = _run(coeffs, sh, 2)
    ref = oshift.shift_coeffs(coeffs, sh, 2)
    assert _rel(got, ref).max() <= TOL


@pytest.mark.parametrize("n", [1, 4, 8, 10, 12])
def test_1d_sizes(n):
    N = 1 << n
    shifts = np.array([0.0, 1.0, N / 2, 0.5, 3.3, -N - 0.75, N / 4, 7.0])
    coeffs = synth.random_signals(300 + n, len(shifts), N)[:, None, :]
    got = _run(coeffs, shifts[:, None, None], 1)
    ref = oshift.shift_coeffs(coeffs, shifts[:, None, None], 1)
    assert _rel(got, ref).max() <= TOL


def test_c2_hdr_32():
    cfg = synth.config("c2")
    light = synth.light_pyramids(cfg.seed, 2, 1, cfg.log2n)
    sh = np.array([[[3.25, 7.5]], [[0.0, 12.0]]])
    got = _run(light, sh, 2)
    ref = oshift.shift_coeffs(light, sh, 2)
    assert _rel(got, ref).max() <= TOL


def test_c3_all_360_frames():
    cfg = synth.config("c3")
    light = synth.light_pyramids(cfg.seed, 1, cfg.faces, cfg.log2n)
    s = synth.c3_shifts(cfg.log2n, 360)
    coeffs = np.broadcast_to(light, (360, cfg.faces, 4 ** cfg.log2n))
    sh = np.broadcast_to(s[:, None, :], (360, cfg.faces, 2))
    got = _run(coeffs, sh, 2)
    ref = oshift.shift_coeffs(coeffs, sh, 2)
    assert _rel(got.reshape(360, -1), ref.reshape(360, -1)).max() <= TOL


def test_c5_batch_64_frames_full_and_band():
    cfg = synth.config("c5")
    light = synth.light_pyramids(cfg.seed, cfg.frames, cfg.faces, cfg.log2n)
    s = synth.c5_shifts(cfg.seed, cfg.frames, cfg.log2n)
    sh = np.broadcast_to(s[:, None, :], (cfg.frames, cfg.faces, 2))
    got = _run(light, sh, 2)
    ref = oshift.shift_coeffs(light, sh, 2)
    rel = _rel(got.reshape(cfg.frames, -1), ref.reshape(cfg.frames, -1))
    assert rel.max() <= TOL, rel.max()
    band = _run(light, sh, 2, band=cfg.band_levels)
    np.testing.assert_array_equal(band, got[:, :, :cfg.k_face])


def test_dyadic_and_identity_faces_mixed_in_one_batch():
    n, N = 8, 256
    shifts = [(0, 0), (256, 512), (128, 0), (64, 192), (4, 8), (0, 2), (1, 0), (0.5, 0), (32, 32.25)]
    B = len(shifts)
    coeffs = synth.light_pyramids(7, B, 1, n)
    sh = np.array(shifts, dtype=np.float64)[:, None, :]
    got = _run(coeffs, sh, 2)
    ref = oshift.shift_coeffs(coeffs, sh, 2)
    assert _rel(got, ref).max() <= TOL
    np.testing.assert_array_equal(got[0], coeffs[0].astype(np.float64))   # identity is a bit-exact copy
    np.testing.assert_array_equal(got[1], coeffs[1].astype(np.float64))


@pytest.mark.parametrize("band", [0, 1, 3, 5])
def test_band_prefix(band):
    n = 6
    coeffs = synth.light_pyramids(9, 3, 6, n)
    sh = np.random.default_rng(4).uniform(-30, 30, size=(3, 6, 2))
    sh[1] = np.round(sh[1])                   # integer (partly dyadic) shifts
    got = _run(coeffs, sh, 2, band=band)
    ref = oshift.shift_coeffs(coeffs, sh, 2, band_levels=band)
    assert got.shape == ref.shape
    assert _rel(got.reshape(-1), ref.reshape(-1)) <= TOL


def test_large_face_global_coarse_path():
    """log2n = 10 and 12: tile-root level c = 7 and 9 > 6 takes the global-memory coarse finish."""
    for n in (10, 12):
        coeffs = synth.light_pyramids(13 + n, 1, 1, n)
        sh = np.array([[[123.375, -77.5]]])
        got = _run(coeffs, sh, 2)
        ref = oshift.shift_coeffs(coeffs, sh, 2)
        assert _rel(got.reshape(-1), ref.reshape(-1)) <= TOL


def test_many_faces_chunked_launches():
    """More than 512 faces per call: several chunked launches, one workspace."""
    n = 4
    B, F = 100, 6
    coeffs = synth.random_signals(15, B * F, 256).reshape(B, F, 256)
    sh = np.random.default_rng(16).uniform(-20, 20, size=(B, F, 2))
    got = _run(coeffs, sh, 2)
    ref = oshift.shift_coeffs(coeffs, sh, 2)
    assert _rel(got, ref).max() <= TOL


def test_deterministic_repeat():
    coeffs = synth.light_pyramids(17, 4, 6, 7)
    sh = np.random.default_rng(18).uniform(0, 128, size=(4, 6, 2))
    a = _run(coeffs, sh, 2)
    b = _run(coeffs, sh, 2)
    np.testing.assert_array_equal(a, b)


def test_launch_count_reported():
    _run(synth.random_signals(19, 1, 64)[None], np.array([[[0.5, 0.5]]]), 2)
    assert _hs().last_launch_count() >= 1


@pytest.mark.parametrize("ndim,n", [(2, 6), (2, 8), (1, 5)])
def test_unaligned_pointers_are_refused(ndim, n):
    """The ABI contract (include/haarshift.h): in / out 16-byte aligned, HS_ERR_ALIGNMENT otherwise
    -- checked before any launch.  (Faces inside a batch may sit at 8-byte offsets: 1D N = 2,
    test_1d_sizes; the kernels take their scalar staging path there.)"""
    import torch
    hs = _hs()
    from paper_1705_07272_b200._lib import HaarShiftError
    N = 1 << n
    K = N * N if ndim == 2 else N
    B, F = 2, 2
    sh = np.full((B, F, ndim), 0.25)
    buf = torch.zeros(B * F * K + 1, device="cuda")
    x = buf[1:].view(B, F, K)
    with pytest.raises(HaarShiftError, match="ALIGNMENT"):
        hs.haar_shift_coeffs(x, sh, ndim)
    obuf = torch.zeros(B * F * K + 1, device="cuda")
    with pytest.raises(HaarShiftError, match="ALIGNMENT"):
        hs.haar_shift_coeffs(buf[:-1].view(B, F, K), sh, ndim, out=obuf[1:].view(B, F, K))
