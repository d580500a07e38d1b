"""Triple-product relight on the GPU (-m gpu).

* haar_pack_qtree against the layout written out here from include/haarshift.h: the 63 detail
  slots of every chunk bit-exact, the cell-mean slot against the fp64 mean of the reconstruction;
* relight_vertices_triple against the fp64 oracle (oracle.relight.relight_triple: the pixel-domain
  triple integral), rel-L2 <= 1e-5, on the tensor-core path (batch % 64 == 0) and the CUDA-core
  path, for k = 3..6, ragged vertex counts, one and six faces;
* the c5t configuration's shapes (64 shifted frames, 6 x 1024 coefficients) on a vertex subset,
  in the launch configuration bench.py times.
"""
import numpy as np
import pytest

import synth
from oracle import haar
from oracle import relight as orelight

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _t(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _rel(got, ref):
    return np.linalg.norm(got - ref) / np.linalg.norm(ref)


def _idx(l, t, i, j):
    return 4 ** l * (1 + t) + i * 2 ** l + j


def _pack_ref(rows, faces, k):
    """qtree layout from its definition in include/haarshift.h (fp64 cell means)."""
    rows = np.asarray(rows, dtype=np.float64)
    R, kf, r = rows.shape[0], 4 ** k, k - 3
    out = np.zeros((R, faces, kf))
    for v in range(R):
        for f in range(faces):
            src = rows[v, f * kf:(f + 1) * kf]
            means = haar.inverse2d(src[:4 ** r]).reshape(-1) if r > 0 else src[:1]
            for ci in range(2 ** r):
                for cj in range(2 ** r):
                    c = ci * 2 ** r + cj
                    o = out[v, f, 64 * c:64 * (c + 1)]
                    for q in range(4):
                        i1, j1 = 2 * ci + (q >> 1), 2 * cj + (q & 1)
                        for p in range(4):
                            i2, j2 = 2 * i1 + (p >> 1), 2 * j1 + (p & 1)
                            for t in range(3):
                                o[15 * q + 3 * p + t] = src[_idx(r + 2, t, i2, j2)]
                        for t in range(3):
                            o[15 * q + 12 + t] = src[_idx(r + 1, t, i1, j1)]
                    for t in range(3):
                        o[60 + t] = src[_idx(r, t, ci, cj)]
                    o[63] = means[c]
    return out.reshape(R, faces * kf)


@pytest.mark.parametrize("k,faces,stride", [(3, 1, 64), (4, 6, 256), (5, 2, 4096), (6, 1, 4096)])
def test_pack_qtree_layout(k, faces, stride):
    import torch
    import paper_1705_07272_b200 as hs
    rows = 7
    src = synth.transfer_rows(41, 0, rows, faces, stride, synth.STREAM_BRDF).reshape(rows, faces, stride)
    got = hs.haar_pack_qtree(_t(src), k).cpu().numpy()
    torch.cuda.synchronize()
    kf = 4 ** k
    ref = _pack_ref(src[:, :, :kf].reshape(rows, faces * kf), faces, k)
    detail = (np.arange(faces * kf) % 64) != 63
    np.testing.assert_array_equal(got[:, detail], ref[:, detail].astype(np.float32))
    np.testing.assert_allclose(got[:, ~detail], ref[:, ~detail], rtol=2e-6, atol=1e-7)


def fill_shading(out, r0, faces, kf, seed, stream):
    """device twin of synth.shading_rows (same fp32 operations after hs_fill_transfer)"""
    import paper_1705_07272_b200 as hs
    hs.hs_fill_transfer(out, r0, faces, kf, seed, stream)
    sc = out[:, ::kf] * 0.5 + 0.5
    out.mul_(0.25)
    out[:, ::kf] = sc


def test_shading_rows_device_twin_bit_exact():
    import torch
    out = torch.empty((33, 6 * 1024), dtype=torch.float32, device="cuda")
    fill_shading(out, 1234, 6, 1024, 99, synth.STREAM_VIS)
    np.testing.assert_array_equal(out.cpu().numpy(), synth.shading_rows(99, 1234, 33, 6, 1024, synth.STREAM_VIS))


def _run(k, faces, V, B, light_log2n=None, seed=50):
    import torch
    import paper_1705_07272_b200 as hs
    kf = 4 ** k
    rho = synth.transfer_rows(seed, 0, V, faces, kf, synth.STREAM_BRDF)
    vis = synth.transfer_rows(seed, 0, V, faces, kf, synth.STREAM_VIS)
    n = light_log2n or k
    L = synth.light_pyramids(seed + 1, B, faces, n)
    rq = hs.haar_pack_qtree(_t(rho).view(V, faces, kf), k)
    vq = hs.haar_pack_qtree(_t(vis).view(V, faces, kf), k)
    R = hs.relight_vertices_triple(rq, vq, _t(L), faces, kf)
    torch.cuda.synchronize()
    return R.cpu().numpy(), orelight.relight_triple(rho, vis, L, faces, kf)


@pytest.mark.parametrize("k,faces,V,B", [(3, 1, 257, 64), (4, 6, 300, 64), (5, 6, 1000, 64), (5, 6, 333, 128),
                                         (6, 1, 200, 64), (5, 1, 1, 64), (4, 2, 150, 1024)])
def test_triple_tensor_core_parity(k, faces, V, B):
    got, ref = _run(k, faces, V, B)
    assert _rel(got, ref) <= TOL


@pytest.mark.parametrize("k,faces,V,B", [(3, 1, 129, 1), (4, 6, 300, 3), (5, 6, 250, 8), (5, 2, 77, 13),
                                         (5, 6, 100, 100)])
def test_triple_cuda_core_parity(k, faces, V, B):
    got, ref = _run(k, faces, V, B)
    assert _rel(got, ref) <= TOL


def test_triple_light_band_of_full_pyramids():
    """light stride 4^n > k_face: the band is the prefix of each full shifted pyramid"""
    got, ref = _run(5, 6, 400, 64, light_log2n=7)
    assert _rel(got, ref) <= TOL


def test_triple_unit_visibility_equals_double_product():
    """V = 1 (scaling only): the triple product is the double product of relight_vertices"""
    import torch
    import paper_1705_07272_b200 as hs
    k, faces, V, B = 5, 6, 500, 64
    kf = 4 ** k
    rho = synth.transfer_rows(60, 0, V, faces, kf, synth.STREAM_BRDF)
    one = np.zeros_like(rho)
    one[:, ::kf] = 1.0
    L = synth.light_pyramids(61, B, faces, k)
    rq = hs.haar_pack_qtree(_t(rho).view(V, faces, kf), k)
    oq = hs.haar_pack_qtree(_t(one).view(V, faces, kf), k)
    R3 = hs.relight_vertices_triple(rq, oq, _t(L), faces, kf).cpu().numpy()
    R2 = hs.relight_vertices(_t(rho), _t(L), faces, kf).cpu().numpy()
    torch.cuda.synchronize()
    ref = orelight.relight(rho, L, faces, kf)
    assert _rel(R3, ref) <= TOL and _rel(R2, ref) <= TOL


def test_triple_c5t_shape_subset():
    """c5t launch configuration: 64 frames of 6 x 256^2 pyramids shifted in the Haar domain (band
    k = 5), BRDF and visibility (synth.shading_rows recipe) generated on the device and packed;
    200k vertices, sampled rows checked against the oracle (shift and triple product both from
    the oracle)."""
    import torch
    import paper_1705_07272_b200 as hs
    from oracle import shift as oshift
    cfg = synth.config("c5t")
    V, F, k, kf, n = 200_000, cfg.faces, cfg.band_levels, cfg.k_face, cfg.log2n
    B = cfg.frames
    light = synth.light_pyramids(cfg.seed, 4, F, n)                       # 4 distinct maps, 64 frames
    frames = np.ascontiguousarray(light[np.arange(B) % 4])
    shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
    band = hs.haar_shift_coeffs(_t(frames), shifts, 2, k)
    tmp = torch.empty((20_000, F * kf), dtype=torch.float32, device="cuda")
    rq = torch.empty((V, F * kf), dtype=torch.float32, device="cuda")
    vq = torch.empty_like(rq)
    for r0 in range(0, V, 20_000):
        fill_shading(tmp, r0, F, kf, cfg.seed, synth.STREAM_BRDF)
        hs.haar_pack_qtree(tmp.view(-1, F, kf), k, out=rq[r0:r0 + 20_000])
        fill_shading(tmp, r0, F, kf, cfg.seed, synth.STREAM_VIS)
        hs.haar_pack_qtree(tmp.view(-1, F, kf), k, out=vq[r0:r0 + 20_000])
    R = hs.relight_vertices_triple(rq, vq, band, F, kf)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, 1, V - 1], np.random.default_rng(5).integers(0, V, 29)]))
    got = R.cpu().numpy()[rows]
    band_ref = np.stack([np.stack([oshift.shift_coeffs2d(frames[b, f], *shifts[b, f])[:kf] for f in range(F)])
                         for b in range(B)])
    ref = np.concatenate([orelight.relight_triple(synth.shading_rows(cfg.seed, v, 1, F, kf, synth.STREAM_BRDF),
                                                  synth.shading_rows(cfg.seed, v, 1, F, kf, synth.STREAM_VIS),
                                                  band_ref, F, kf) for v in rows])
    assert _rel(got, ref) <= TOL
