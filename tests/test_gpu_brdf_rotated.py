"""The paper's shading composed on the GPU (-m gpu): the BRDF rotated per vertex normal (row f1),
then the triple product with light and visibility (row f3) -- relight_vertices_brdf_rotated
(R28).

Two references, both composed from the fp64 oracle only:
* the paper's algorithm step by step -- oracle.rotate.rotate_coeffs_chain per vertex, then
  oracle.relight.relight_triple (the pixel-domain triple integral): the GPU must equal it within
  rel-L2 1e-5 (a regression check that the composition runs the algorithm, incl. the chunking);
* the spatial ground truth -- oracle.rotate.rotate_coeffs (bilinear resampling at the rotated
  angles), then relight_triple: accuracy, reported as rel-L2, must be as good as the
  algorithm's own (the chain oracle's) to 1e-5 and shrink with the resolution (first-order chain
  rule).
"""
import numpy as np
import pytest

import synth
from oracle import relight as orelight
from oracle import rotate as orot

pytestmark = pytest.mark.gpu


def _normals(seed, V):
    v = np.random.default_rng(seed).normal(size=(V, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    theta = np.arccos(np.clip(v[:, 1], -1.0, 1.0))
    phi = np.mod(np.arctan2(v[:, 0], v[:, 2]), 2.0 * np.pi)
    return np.stack([theta, phi], axis=1)


def _case(seed, n, k, V, B):
    brdf = synth.smooth_sphere_maps(seed, 1, n)[0]
    kf = 4 ** k
    vis = synth.shading_rows(seed, 0, V, 1, kf, synth.STREAM_VIS)
    light = synth.light_pyramids(seed, B, 1, n)[:, 0, :]
    return brdf, vis, light, _normals(seed, V)


def _gpu(brdf, vis, light, normals, k):
    import torch
    import paper_1705_07272_b200 as hs
    V = vis.shape[0]
    dv = torch.from_numpy(np.ascontiguousarray(vis, dtype=np.float32)).cuda()
    vq = hs.haar_pack_qtree(dv.view(V, 1, 4 ** k), k).view(V, 4 ** k)
    R = hs.relight_vertices_brdf_rotated(torch.from_numpy(brdf).cuda(), normals, vq,
                                         torch.from_numpy(np.ascontiguousarray(light)).cuda(), k)
    torch.cuda.synchronize()
    return R.cpu().numpy().astype(np.float64)


def _reference(brdf, vis, light, normals, k, rotate, rows=None):
    kf = 4 ** k
    rows = np.arange(vis.shape[0]) if rows is None else np.asarray(rows)
    rho = np.stack([rotate(brdf.astype(np.float64), float(normals[v, 0]), float(normals[v, 1]))[:kf] for v in rows])
    return orelight.relight_triple(rho, vis[rows].astype(np.float64), light[:, None, :].astype(np.float64), 1, kf)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("B", [64, 3])
def test_composed_equals_the_algorithm(B):
    """tensor-core (B = 64) and CUDA-core (B = 3) triple products; 257 vertices = 2 full 128-row
    tiles + a ragged one"""
    brdf, vis, light, nrm = _case(1701, 4, 3, 257, B)
    got = _gpu(brdf, vis, light, nrm, 3)
    ref = _reference(brdf, vis, light, nrm, 3, orot.rotate_coeffs_chain)
    assert _rel(got, ref) <= 1e-5


def test_composed_across_chunks():
    """4096-vertex rotation chunks: vertices on both sides of the boundary, sampled"""
    V = 4096 + 300
    brdf, vis, light, nrm = _case(1702, 4, 3, V, 64)
    got = _gpu(brdf, vis, light, nrm, 3)
    rows = np.r_[0:8, 4088:4104, V - 8:V, np.random.default_rng(3).integers(0, V, 16)]
    ref = _reference(brdf, vis, light, nrm, 3, orot.rotate_coeffs_chain, rows)
    assert _rel(got[rows], ref) <= 1e-5


def test_zero_elevation_is_the_plain_triple_product():
    """theta_N = phi_N = 0: no rotation -- the composed call equals relight_vertices_triple of the
    unrotated BRDF"""
    import torch
    import paper_1705_07272_b200 as hs
    n, k, V, B = 5, 4, 200, 64
    brdf, vis, light, _ = _case(1703, n, k, V, B)
    nrm = np.zeros((V, 2))
    got = _gpu(brdf, vis, light, nrm, k)
    kf = 4 ** k
    rho = np.broadcast_to(brdf[:kf], (V, kf)).astype(np.float64)
    ref = orelight.relight_triple(rho, vis.astype(np.float64), light[:, None, :].astype(np.float64), 1, kf)
    assert _rel(got, ref) <= 1e-5
    # and bitwise-stable against the two-call form
    dev = torch.device("cuda")
    rq = hs.haar_pack_qtree(torch.from_numpy(np.ascontiguousarray(np.broadcast_to(brdf, (V, brdf.size)))).to(dev)
                            .view(V, 1, brdf.size), k).view(V, kf)
    vq = hs.haar_pack_qtree(torch.from_numpy(vis).to(dev).view(V, 1, kf), k).view(V, kf)
    two = hs.relight_vertices_triple(rq, vq, torch.from_numpy(np.ascontiguousarray(light)).to(dev).view(B, 1, -1), 1, kf)
    torch.cuda.synchronize()
    assert _rel(got, two.cpu().numpy().astype(np.float64)) <= 1e-6


def test_accuracy_against_the_spatial_rotation():
    """rel-L2 of the radiance against rotating the BRDF in the spatial domain: the GPU's error equals
    the algorithm's own (chain oracle) and shrinks with N (first order in the pixel size)"""
    errs = []
    for n in (4, 5):
        brdf, vis, light, nrm = _case(1704, n, 3, 48, 64)
        got = _gpu(brdf, vis, light, nrm, 3)
        spatial = _reference(brdf, vis, light, nrm, 3, orot.rotate_coeffs)
        chain = _reference(brdf, vis, light, nrm, 3, orot.rotate_coeffs_chain)
        e_gpu, e_alg = _rel(got, spatial), _rel(chain, spatial)
        assert abs(e_gpu - e_alg) <= 1e-5 * max(1.0, e_alg) + 1e-6
        errs.append(e_gpu)
    assert errs[1] < errs[0]


def test_composed_edge_normals_and_full_band():
    """normals at the poles, on the equator at phi = 0 and pi, and just inside the 2 pi seam; the
    band equal to the whole map (log2k = log2n); 130 vertices (a ragged 128-row tile)"""
    n = k = 4
    brdf, vis, light, nrm = _case(1705, n, k, 130, 64)
    edge = np.array([[0.0, 0.0], [np.pi, 0.0], [np.pi / 2, 0.0], [np.pi / 2, np.pi], [1e-9, 2 * np.pi - 1e-9],
                     [np.pi - 1e-9, 1e-9], [np.pi / 4, 3 * np.pi / 2]])
    nrm[:len(edge)] = edge
    got = _gpu(brdf, vis, light, nrm, k)
    ref = _reference(brdf, vis, light, nrm, k, orot.rotate_coeffs_chain)
    assert _rel(got, ref) <= 1e-5
    assert _rel(got[:len(edge)], ref[:len(edge)]) <= 1e-5
