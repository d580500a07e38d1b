"""Sparse-transfer relight on the GPU (-m gpu): the seeded sparse generator
is bit-exact with synth, and the gather relight matches the fp64 oracle (rel-L2 <= 1e-5)."""
import numpy as np
import pytest

import synth
from oracle import relight as orelight

pytestmark = pytest.mark.gpu
TOL = 1e-5


def test_fill_sparse_bit_exact():
    import torch
    import paper_1705_07272_b200 as hs
    for faces, n, ks, dl, r0, rows in [(6, 8, 256, 2, 0, 100), (6, 5, 100, 1, 12345, 33), (1, 3, 20, 0, 7, 9)]:
        idx = torch.empty((rows, ks), dtype=torch.int32, device="cuda")
        val = torch.empty((rows, ks), dtype=torch.float32, device="cuda")
        hs.hs_fill_sparse_transfer(idx, val, r0, faces, n, dl, 77)
        i_ref, v_ref = synth.sparse_transfer_rows(77, r0, rows, faces, n, ks, dl)
        np.testing.assert_array_equal(idx.cpu().numpy(), i_ref)
        np.testing.assert_array_equal(val.cpu().numpy(), v_ref)


@pytest.mark.parametrize("B", [1, 7, 64, 100])
def test_sparse_relight_parity(B):
    import torch
    import paper_1705_07272_b200 as hs
    faces, n, ks, V = 6, 6, 200, 777
    idx, val = synth.sparse_transfer_rows(78, 0, V, faces, n, ks)
    light = synth.light_pyramids(79, B, faces, n)
    R = hs.relight_vertices_sparse(torch.from_numpy(idx).cuda(), torch.from_numpy(val).cuda(),
                                   torch.from_numpy(light).cuda())
    torch.cuda.synchronize()
    ref = orelight.relight_sparse(idx, val, light.reshape(B, -1))
    assert np.linalg.norm(R.cpu().numpy() - ref) / np.linalg.norm(ref) <= TOL


def test_sparse_relight_after_shift_c5_shape_subset():
    """c5 shapes: 64 frames of 6 x 256^2 shifted pyramids, K_s = 256 full-resolution coefficients,
    a 2000-vertex subset of the 1M-vertex matrix."""
    import torch
    import paper_1705_07272_b200 as hs
    cfg = synth.config("c5")
    B, V, ks = 64, 2000, 256
    light = synth.light_pyramids(cfg.seed, B, cfg.faces, cfg.log2n)
    sh = np.broadcast_to(synth.c5_shifts(cfg.seed, B, cfg.log2n)[:, None, :], (B, cfg.faces, 2)).copy()
    shifted = hs.haar_shift_coeffs(torch.from_numpy(light).cuda(), sh, 2)
    idx = torch.empty((V, ks), dtype=torch.int32, device="cuda")
    val = torch.empty((V, ks), dtype=torch.float32, device="cuda")
    hs.hs_fill_sparse_transfer(idx, val, 500000, cfg.faces, cfg.log2n, 2, cfg.seed)
    R = hs.relight_vertices_sparse(idx, val, shifted)
    torch.cuda.synchronize()
    ref = orelight.relight_sparse(idx.cpu().numpy(), val.cpu().numpy(), shifted.cpu().numpy().reshape(B, -1))
    assert np.linalg.norm(R.cpu().numpy() - ref) / np.linalg.norm(ref) <= TOL


@pytest.mark.parametrize("faces,n,B,ks", [(6, 6, 64, 150), (6, 2, 3, 150), (24, 4, 70, 152), (1, 8, 128, 256),
                                          (2, 5, 64, 33)])
def test_sparse_shapes(faces, n, B, ks):
    """full 64-frame blocks (vectorised path: K_s % 4 == 0) and ragged ones (scalar path), one and
    many faces, B = 70 mixing both"""
    import torch
    import paper_1705_07272_b200 as hs
    V = 555
    idx, val = synth.sparse_transfer_rows(80, 0, V, faces, n, ks, 1 if faces > 6 else min(2, n - 1))
    light = synth.light_pyramids(81, B, faces, n)
    R = hs.relight_vertices_sparse(torch.from_numpy(idx).cuda(), torch.from_numpy(val).cuda(),
                                   torch.from_numpy(light).cuda()).cpu().numpy()
    ref = orelight.relight_sparse(idx, val, light.reshape(B, -1))
    assert np.linalg.norm(R - ref) / np.linalg.norm(ref) <= TOL


def test_sparse_host_pipeline_matches_device_calls():
    """ShiftSparseRelightPipeline (host buffers, chunked D2H under the next chunk's relight) returns
    exactly the device path's radiance, step after step"""
    import torch
    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200.pipeline import ShiftSparseRelightPipeline
    n, F, B, V, ks = 5, 6, 64, 1001, 128
    idx = torch.empty((V, ks), dtype=torch.int32, device="cuda")
    val = torch.empty((V, ks), dtype=torch.float32, device="cuda")
    hs.hs_fill_sparse_transfer(idx, val, 0, F, n, 2, 33)
    pipe = ShiftSparseRelightPipeline(idx, val, F, n, B, chunks=3)
    outs, refs = [], []
    for step in range(3):
        light = synth.light_pyramids(50 + step, B, F, n)
        sh = np.random.default_rng(step).uniform(0, 32, size=(B, F, 2))
        lh = torch.from_numpy(light).pin_memory()
        rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        pipe.step(lh, sh, rh)
        outs.append(rh)
        s = hs.haar_shift_coeffs(torch.from_numpy(light).cuda(), sh, 2)
        refs.append(hs.relight_vertices_sparse(idx, val, s).cpu())
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)
