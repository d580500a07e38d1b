"""Coarse-start shift (R23) on the GPU (-m gpu):
parity with the oracle's definition (the shift of the level-L approximation), exactness for shifts
that are multiples of 2**(n-L), and the accuracy-vs-start-level study against the exact shift."""
import numpy as np
import pytest

import synth
from oracle import shift as oshift

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _run(coeffs, shifts, L, band=None):
    import torch
    import paper_1705_07272_b200 as hs
    out = hs.haar_shift_coeffs_coarse(torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float32)).cuda(),
                                      shifts, L, band)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,L", [(5, 3), (6, 4), (8, 5), (8, 6), (8, 8)])
def test_coarse_parity_with_oracle_definition(n, L):
    B, F = 4, 6
    light = synth.light_pyramids(50 + n + L, B, F, n)
    sh = np.random.default_rng(L).uniform(-40, 40, size=(B, F, 2))
    got = _run(light, sh, L)
    for b in range(B):
        for f in range(F):
            ref = oshift.shift_coeffs_coarse2d(light[b, f], L, *sh[b, f])
            assert _rel(got[b, f], ref) <= TOL


def test_coarse_exact_for_multiples_of_cell():
    n, L = 8, 5
    light = synth.light_pyramids(60, 3, 1, n)
    sh = np.array([[[8.0, 16.0]], [[-24.0, 40.0]], [[0.0, 248.0]]])     # multiples of 2**(n-L) = 8
    got = _run(light, sh, L)
    ref = oshift.shift_coeffs(light, sh, 2, band_levels=L)
    assert _rel(got.reshape(-1), ref.reshape(-1)) <= TOL


def test_coarse_accuracy_study_vs_exact():
    """PSNR of the relight band (levels < 5) from start levels 5..8 against the exact shift: it
    improves monotonically with the start level and is exact at L = n (the paper's "slight loss
    of accuracy" for coarser starts)."""
    n, band = 8, 5
    light = synth.light_pyramids(61, 8, 6, n)
    sh = synth.c5_shifts(61, 8, n)
    sh = np.broadcast_to(sh[:, None, :], (8, 6, 2)).copy()
    exact = oshift.shift_coeffs(light, sh, 2, band_levels=band)
    peak = np.abs(exact).max()
    psnr = []
    for L in (5, 6, 7, 8):
        got = _run(light, sh, L, band)
        mse = np.mean((got - exact) ** 2)
        psnr.append(10 * np.log10(peak ** 2 / max(mse, 1e-300)))
    assert all(psnr[i] <= psnr[i + 1] + 1e-6 for i in range(3)), psnr
    assert psnr[-1] > 100.0, psnr
