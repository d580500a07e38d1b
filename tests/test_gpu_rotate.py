"""Rotation of lat-long maps in the Haar domain on the GPU (-m gpu).

Accuracy of the method -- the headline for f1, as the paper reports it (PSNR against rotating in
the spatial domain):
* alpha = 0 reproduces the input (rel-L2 <= 1e-5) and an integer azimuth is the exact column
  permutation of the spatial oracle (rel-L2 <= 1e-5) -- the exact parts;
* for alpha != 0 the GPU result is compared, as PSNR, with the spatial ground truth (oracle.rotate:
  bilinear resampling at the rotated angles) and with the analytic rotation of the smooth maps.
  The floors are not measured values: the GPU must be as accurate as the paper's algorithm itself
  (oracle.rotate.rotate_coeffs_chain, fp64) to within 0.1 dB, and its PSNR against the analytic
  rotation must rise with the resolution (the chain rule is first order in the pixel size).

Regression check: the GPU equals rotate_coeffs_chain (the paper's algorithm step by step in fp64,
each stage pinned in tests/test_oracle_rotate.py) within rel-L2 1e-5, for smooth and white-noise
maps, random elevations (poles crossed) and azimuths, N = 2 .. 2048 (the DC's level cap binds at
N >= 128).  That agreement shows the kernels implement the algorithm; it is not an accuracy claim.
"""
import math

import numpy as np
import pytest

import synth
from oracle import rotate as orot

pytestmark = pytest.mark.gpu


def _rot(c, ang):
    import torch
    import paper_1705_07272_b200 as hs
    out = hs.haar_rotate_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(), ang)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n", [3, 5, 6])
def test_identity(n):
    c = synth.smooth_sphere_maps(11, 5, n)
    got = _rot(c, np.zeros((5, 2)))
    assert _rel(got, c) <= 1e-5


@pytest.mark.parametrize("n,k", [(5, 3), (6, 17), (7, 64)])
def test_integer_azimuth_is_exact(n, k):
    N = 1 << n
    c = synth.smooth_sphere_maps(12, 3, n)
    ang = np.array([[0.0, k * 2 * math.pi / N], [0.0, -k * 2 * math.pi / N], [0.0, 0.5 * 2 * math.pi / N]])
    got = _rot(c, ang)
    for b in range(3):
        ref = orot.rotate_coeffs(c[b], *ang[b])
        assert _rel(got[b], ref) <= 1e-5


def _truth(seed, k, n, alpha, beta):
    """cell means of the exactly rotated analytic map (Gauss-Legendre 4 x 4 per pixel)"""
    N = 1 << n
    g, w = np.polynomial.legendre.leggauss(4)
    th = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * np.pi / N
    ph = (np.arange(N)[:, None] + 0.5 + 0.5 * g[None, :]) * 2 * np.pi / N - beta   # f'(phi) = f(phi - beta)
    T, P = np.broadcast_arrays(th[:, None, :, None], ph[None, :, None, :])
    Th, Ph = orot.rotated_angles(T, P, alpha)
    vals = synth.smooth_sphere_eval(seed, k, Th, Ph)
    return np.einsum("rcab,a,b->rc", vals, w, w) / 4.0


def _psnr_pix(a, ref):
    return 10 * np.log10(np.abs(ref).max() ** 2 / np.mean((a - ref) ** 2))


def test_psnr_against_spatial_and_analytic_ground_truth():
    """GPU chain-rule rotation vs the spatial oracle (the paper's ground truth) and vs the
    analytic rotation of the smooth maps.  Floors from principle, not from measurements: within
    0.1 dB of the fp64 algorithm (rotate_coeffs_chain) against the same truths, and rising with N"""
    from oracle import haar
    med_gt = {}
    for n in (5, 6, 7, 8):
        c = synth.smooth_sphere_maps(13, 6, n)
        ang = synth.rotation_angles(14, 6)
        got = _rot(c, ang)
        p_or, p_gt, q_or, q_gt = [], [], [], []
        for b in range(6):
            ref = orot.rotate_coeffs(c[b], *ang[b])
            chain = orot.rotate_coeffs_chain(c[b], *ang[b])
            truth = _truth(13, b, n, *ang[b])
            p_or.append(orot.psnr(got[b], ref))
            q_or.append(orot.psnr(chain, ref))
            p_gt.append(_psnr_pix(haar.inverse2d(got[b]), truth))
            q_gt.append(_psnr_pix(haar.inverse2d(chain), truth))
        med_gt[n] = float(np.median(p_gt))
        print(f"n={n}: vs spatial oracle GPU min {min(p_or):.1f} median {np.median(p_or):.1f} dB "
              f"(fp64 algorithm min {min(q_or):.1f}) | vs analytic GPU min {min(p_gt):.1f} median "
              f"{np.median(p_gt):.1f} dB (fp64 algorithm median {np.median(q_gt):.1f})")
        for b in range(6):
            assert p_or[b] >= q_or[b] - 0.1 and p_gt[b] >= q_gt[b] - 0.1, (n, b)
    assert med_gt[5] < med_gt[6] < med_gt[7] < med_gt[8]


@pytest.mark.parametrize("n,kind", [(1, "noise"), (2, "noise"), (3, "smooth"), (4, "noise"), (5, "smooth"),
                                    (6, "smooth"), (6, "noise"), (7, "smooth"), (8, "smooth"), (9, "noise"),
                                    (11, "noise")])
def test_parity_with_chain_rule_oracle(n, kind):
    rng = np.random.default_rng(100 + n)
    B = 6 if n <= 9 else 3
    if kind == "smooth":
        c = synth.smooth_sphere_maps(20 + n, B, n)
    else:
        from oracle import haar
        c = np.stack([haar.forward2d(m) for m in synth.random_signals(30 + n, B, 4 ** n).reshape(B, 1 << n, 1 << n)])
    ang = np.column_stack([rng.uniform(-math.pi, math.pi, B), rng.uniform(-math.pi, math.pi, B)])
    ang[0] = (math.pi, 0.3)           # exact flip
    ang[1] = (1e-3, 0.0)              # near identity
    got = _rot(c, ang)
    for b in range(B):
        ref = orot.rotate_coeffs_chain(c[b], *ang[b])
        err = _rel(got[b], ref)
        print(n, kind, b, ang[b], err)
        assert err <= 1e-5, (n, kind, b, ang[b], err)


def test_rotate_host_pipeline_matches_device_call():
    import torch
    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200.pipeline import RotatePipeline
    n, B = 5, 37
    pipe = RotatePipeline(B, n, torch.device("cuda"), chunks=3)
    for step in range(2):
        c = synth.smooth_sphere_maps(60 + step, B, n)
        ang = synth.rotation_angles(61 + step, B)
        xh = torch.from_numpy(c).pin_memory()
        yh = torch.empty((B, 4 ** n), dtype=torch.float32).pin_memory()
        pipe.step(xh, ang, yh).synchronize()
        ref = hs.haar_rotate_coeffs(torch.from_numpy(c).cuda(), ang).cpu()
        assert torch.equal(yh, ref)
