"""GPU parity of relight_vertices / relight_vertices_shifted / hs_fill_transfer against the fp64
oracle and the seeded generator (-m gpu).  Gate: relative L2 <= 1e-5 per radiance tensor."""
import numpy as np
import pytest

import synth
from oracle import relight as orelight
from oracle import shift as oshift

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _t(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _rel(got, ref):
    return np.linalg.norm(got - ref) / np.linalg.norm(ref)


def test_fill_transfer_bit_exact():
    import torch
    import paper_1705_07272_b200 as hs
    for faces, kf, r0, rows in [(6, 1024, 0, 300), (6, 16, 12345, 77), (1, 4, 999_999, 5), (6, 4096, 7, 33)]:
        out = torch.empty((rows, faces * kf), dtype=torch.float32, device="cuda")
        hs.hs_fill_transfer(out, r0, faces, kf, synth.SEED_BASE + 5, synth.STREAM_T)
        np.testing.assert_array_equal(out.cpu().numpy(), synth.transfer_rows(synth.SEED_BASE + 5, r0, rows, faces, kf))


@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 6, 7, 8])
def test_gemv_small_batches(B):
    import torch
    import paper_1705_07272_b200 as hs
    faces, kf, V = 6, 256, 1001                       # V odd: row-group tail
    T = synth.transfer_rows(3, 0, V, faces, kf)
    L = synth.light_pyramids(4, B, faces, 4)          # stride 256 = kf
    R = hs.relight_vertices(_t(T), _t(L), faces, kf)
    torch.cuda.synchronize()
    ref = orelight.relight(T, L, faces, kf)
    assert _rel(R.cpu().numpy(), ref) <= TOL


def test_strided_light_band_from_full_pyramids():
    import torch
    import paper_1705_07272_b200 as hs
    faces, kf, V = 6, 64, 513
    T = synth.transfer_rows(5, 0, V, faces, kf)
    L = synth.light_pyramids(6, 3, faces, 5)          # stride 1024 > kf
    R = hs.relight_vertices(_t(T), _t(L), faces, kf)
    torch.cuda.synchronize()
    assert _rel(R.cpu().numpy(), orelight.relight(T, L, faces, kf)) <= TOL


@pytest.mark.parametrize("B", [9, 13, 64, 128, 1024])
def test_gemm_batches(B):
    import torch
    import paper_1705_07272_b200 as hs
    faces, kf, V = 6, 1024, 3000
    T = synth.transfer_rows(7, 0, V, faces, kf)
    L = synth.light_pyramids(8, B, faces, 5)
    R = hs.relight_vertices(_t(T), _t(L), faces, kf)
    torch.cuda.synchronize()
    assert _rel(R.cpu().numpy(), orelight.relight(T, L, faces, kf)) <= TOL


def test_c3_relight_one_frame():
    import torch
    import paper_1705_07272_b200 as hs
    cfg = synth.config("c3")
    T = torch.empty((cfg.vertices, cfg.faces * cfg.k_face), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, cfg.faces, cfg.k_face, cfg.seed, synth.STREAM_T)
    light = synth.light_pyramids(cfg.seed, 1, cfg.faces, cfg.log2n)
    s = synth.c3_shifts(cfg.log2n, 360)[[37]]
    sh = np.broadcast_to(s[:, None, :], (1, cfg.faces, 2))
    shifted, R = hs.shift_and_relight(_t(light), sh, T, cfg.faces, cfg.k_face, cfg.log2n)
    torch.cuda.synchronize()
    Lref = oshift.shift_coeffs(light, sh, 2)
    ref = orelight.relight(T.cpu().numpy(), Lref, cfg.faces, cfg.k_face)
    assert _rel(R.cpu().numpy(), ref) <= TOL


def test_relight_shifted_small():
    import torch
    import paper_1705_07272_b200 as hs
    n, F, V = 5, 6, 300
    L = synth.light_pyramids(21, 1, F, n)[0]
    T = synth.transfer_rows(22, 0, V, F, 4 ** n)
    sv = synth.c4_vertex_shifts(23, V, n)
    sv[:5] = [[0, 0], [32, 0], [16, 8], [1, 1], [0.5, 0]]          # identity / dyadic / integer
    R = hs.relight_vertices_shifted(_t(T), _t(L), _t(sv))
    torch.cuda.synchronize()
    ref = orelight.relight_shifted(T, L, sv.astype(np.float64))
    assert _rel(R.cpu().numpy(), ref) <= TOL


def test_relight_shifted_c4_subset():
    """c4 shape (6 x 128 x 128, full-pyramid transfer), a 200-vertex subset."""
    import torch
    import paper_1705_07272_b200 as hs
    cfg = synth.config("c4")
    V = 200
    L = synth.light_pyramids(cfg.seed, 1, cfg.faces, cfg.log2n)[0]
    T = torch.empty((V, cfg.faces * 4 ** cfg.log2n), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 5000, cfg.faces, 4 ** cfg.log2n, cfg.seed, synth.STREAM_T)
    sv = synth.c4_vertex_shifts(cfg.seed, 6000, cfg.log2n)[5000:5000 + V]
    R = hs.relight_vertices_shifted(T, _t(L), _t(sv))
    torch.cuda.synchronize()
    ref = orelight.relight_shifted(T.cpu().numpy(), L, sv.astype(np.float64))
    assert _rel(R.cpu().numpy(), ref) <= TOL


def test_host_pipeline_matches_device_calls():
    """ShiftRelightPipeline (host buffers, overlapped copies) returns exactly the device path's
    radiance, step after step (double-buffered light, chunked D2H)."""
    import torch
    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200.pipeline import ShiftRelightPipeline
    n, F, B, V, band = 5, 6, 64, 1000, 3
    T = torch.empty((V, F * 4 ** band), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, 4 ** band, 31, synth.STREAM_T)
    pipe = ShiftRelightPipeline(T, F, n, B, band, chunks=3)
    outs, refs = [], []
    for step in range(3):
        light = synth.light_pyramids(40 + step, B, F, n)
        sh = np.random.default_rng(step).uniform(0, 32, size=(B, F, 2))
        lh = torch.from_numpy(light).pin_memory()
        rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        pipe.step(lh, sh, rh)
        outs.append(rh)
        s = hs.haar_shift_coeffs(torch.from_numpy(light).cuda(), sh, 2)
        refs.append(hs.relight_vertices(T, s, F, 4 ** band).cpu())
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)


def test_sharded_host_pipeline_single_rank_matches_device_calls():
    """ShardedShiftRelightPipeline (the N>1 host-buffer step: own frames H2D, band shift, band
    all-gather, chunked relight with per-chunk D2H into a shared page-locked host array), run as
    one rank: bitwise the device calls' radiance, step after step"""
    import torch
    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200 import dist as hsdist
    from paper_1705_07272_b200.pipeline import ShardedShiftRelightPipeline
    n, F, B, V, band = 5, 6, 64, 1000, 3
    T = torch.empty((V, F * 4 ** band), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, 4 ** band, 32, synth.STREAM_T)
    pipe = ShardedShiftRelightPipeline(T, F, n, B, band, V, chunks=3)
    shared = hsdist.SharedHostBuffer((V, B))
    try:
        for step in range(3):
            light = synth.light_pyramids(50 + step, B, F, n)
            sh = np.random.default_rng(10 + step).uniform(0, 32, size=(B, F, 2))
            ev = pipe.step(torch.from_numpy(light).pin_memory(), sh, shared.tensor)
            ev.synchronize()
            s = hs.haar_shift_coeffs(torch.from_numpy(light).cuda(), sh, 2, band)
            ref = hs.relight_vertices(T, s, F, 4 ** band).cpu()
            assert torch.equal(shared.tensor, ref)
    finally:
        shared.close()
