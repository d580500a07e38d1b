"""Range of the split-precision tensor-core relights (-m gpu).

The tcgen05 kernels split T (relight_vertices) and the tripling terms M (relight_vertices_triple)
into fp16 hi/lo pieces.  Their accuracy must not depend on the absolute magnitude of the inputs
(What's weak #2): every 64-k block of every row is scaled by its own power of two
before the split.  These tests scale the transfer far outside fp16's range --
2^-30, 1e-6, 2^14, 2^60 -- and mix magnitudes between rows and between the blocks of one row, and
hold each ROW of radiance (64 frames) to rel-L2 <= 1e-5 against the fp64 oracle, which is
stricter than one rel-L2 over the tensor (tiny rows would vanish in it).
"""
import numpy as np
import pytest

import synth
from oracle import relight as orelight

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _t(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _row_rel(got, ref):
    num = np.linalg.norm(got - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    return float(np.max(num / den))


def _scaled_rows(T, how, rng):
    T = T.astype(np.float64)
    if how == "mixed_rows":                     # every row 1e-8 or 1, at random
        s = np.where(rng.random(T.shape[0]) < 0.5, 1e-8, 1.0)
        return T * s[:, None]
    if how == "mixed_blocks":                   # 64-k blocks of one row at 1e-8 .. 1e4
        nb = T.shape[1] // 64
        s = 10.0 ** rng.integers(-8, 5, size=(T.shape[0], nb))
        return T * np.repeat(s, 64, axis=1)
    if how == "mixed_within_block":             # magnitudes 1e-8 and 1 inside every block
        s = np.where(rng.random(T.shape) < 0.5, 1e-8, 1.0)
        return T * s
    return T * float(how)


CASES = [2.0 ** -30, 1e-6, 2.0 ** 14, 2.0 ** 60, 1e-30, "mixed_rows", "mixed_blocks", "mixed_within_block"]


@pytest.mark.parametrize("how", CASES)
@pytest.mark.parametrize("B", [64, 128])
def test_tc_relight_any_transfer_magnitude(how, B):
    import torch
    import paper_1705_07272_b200 as hs
    faces, kf, V = 6, 1024, 1500                    # 1500 = 11 full 128-row tiles + a ragged tail
    rng = np.random.default_rng(7)
    T = _scaled_rows(synth.transfer_rows(70, 0, V, faces, kf), how, rng).astype(np.float32)
    assert np.all(np.isfinite(T))
    L = synth.light_pyramids(71, B, faces, 5)
    R = hs.relight_vertices(_t(T), _t(L), faces, kf)
    torch.cuda.synchronize()
    ref = orelight.relight(T, L, faces, kf)
    assert _row_rel(R.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("scale", [2.0 ** -40, 1e-6, 2.0 ** 20])
def test_tc_relight_any_light_magnitude(scale):
    """the light's per-frame power of two covers any light magnitude (and a 2^-40-scaled T on top)"""
    import torch
    import paper_1705_07272_b200 as hs
    faces, kf, V, B = 6, 256, 700, 64
    T = (synth.transfer_rows(72, 0, V, faces, kf).astype(np.float64) * 2.0 ** -40).astype(np.float32)
    L = (synth.light_pyramids(73, B, faces, 4).astype(np.float64) * scale).astype(np.float32)
    R = hs.relight_vertices(_t(T), _t(L), faces, kf)
    torch.cuda.synchronize()
    assert _row_rel(R.cpu().numpy(), orelight.relight(T, L, faces, kf)) <= TOL


@pytest.mark.parametrize("rs,vs", [(2.0 ** -30, 1.0), (1e-6, 1e-3), (2.0 ** 14, 2.0 ** 10), (1.0, 2.0 ** -60),
                                   ("mixed_rows", 1.0)])
def test_tc_triple_any_magnitude(rs, vs):
    import torch
    import paper_1705_07272_b200 as hs
    k, faces, V, B = 5, 6, 600, 64
    kf = 4 ** k
    rng = np.random.default_rng(9)
    rho = synth.shading_rows(74, 0, V, faces, kf, synth.STREAM_BRDF)
    vis = synth.shading_rows(74, 0, V, faces, kf, synth.STREAM_VIS)
    rho = _scaled_rows(rho, rs, rng).astype(np.float32)
    vis = (vis.astype(np.float64) * vs).astype(np.float32)
    L = synth.light_pyramids(75, B, faces, k)
    rq = hs.haar_pack_qtree(_t(rho).view(V, faces, kf), k)
    vq = hs.haar_pack_qtree(_t(vis).view(V, faces, kf), k)
    R = hs.relight_vertices_triple(rq, vq, _t(L), faces, kf)
    torch.cuda.synchronize()
    ref = orelight.relight_triple(rho, vis, L, faces, kf)
    assert _row_rel(R.cpu().numpy(), ref) <= TOL
