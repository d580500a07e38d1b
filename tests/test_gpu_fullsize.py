"""Parity at BASELINE.json's full sizes, in the launch configurations bench.py times (-m gpu):
the whole job runs on the device, the fp64 oracle recomputes seeded sampled outputs one by one.

* c5: 64 frames x 6 faces of 256^2 shifted (full pyramids), 1M vertices x 6144 coefficients on
  the tcgen05 relight -- 48 sampled vertices x 64 frames;
* c4: 100k vertices, per-vertex shifts of 6 x 128^2 (39.3 GB of transfer) on the fused kernel --
  12 sampled vertices.
Gate: rel-L2 <= 1e-5 over the sampled outputs.
"""
import numpy as np
import pytest

import synth
from oracle import relight as orelight
from oracle import shift as oshift

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_c5_full_size_sampled_rows():
    import torch
    import paper_1705_07272_b200 as hs
    cfg = synth.config("c5")
    V, F, n, B, kf = cfg.vertices, cfg.faces, cfg.log2n, cfg.frames, cfg.k_face
    T = torch.empty((V, F * kf), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, kf, cfg.seed, synth.STREAM_T)
    light_np = synth.light_pyramids(cfg.seed, B, F, n)
    shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
    shifted, R = hs.shift_and_relight(torch.from_numpy(light_np).cuda(), shifts, T, F, kf, n)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, 127, 128, V - 1], np.random.default_rng(11).integers(0, V, 44)]))
    got = R[torch.from_numpy(rows).cuda()].cpu().numpy()
    del T
    band = oshift.shift_coeffs(light_np, shifts, 2, band_levels=cfg.band_levels)
    ref = np.concatenate([orelight.relight(synth.transfer_rows(cfg.seed, int(v), 1, F, kf), band, F, kf)
                          for v in rows])
    print(f"c5 full size: rel-L2 {_rel(got, ref):.3e}")
    assert _rel(got, ref) <= TOL


def test_c4_full_size_sampled_vertices():
    import torch
    import paper_1705_07272_b200 as hs
    cfg = synth.config("c4")
    V, F, n = cfg.vertices, cfg.faces, cfg.log2n
    K = F * 4 ** n
    T = torch.empty((V, K), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, 4 ** n, cfg.seed, synth.STREAM_T)
    L = synth.light_pyramids(cfg.seed, 1, F, n)[0]
    sv = synth.c4_vertex_shifts(cfg.seed, V, n)
    R = hs.relight_vertices_shifted(T, torch.from_numpy(L).cuda(), torch.from_numpy(sv).cuda())
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, V - 1], np.random.default_rng(12).integers(0, V, 10)]))
    got = R.cpu().numpy()[rows]
    del T
    ref = np.array([orelight.relight_shifted(synth.transfer_rows(cfg.seed, int(v), 1, F, 4 ** n), L,
                                             sv[v:v + 1].astype(np.float64))[0] for v in rows])
    print(f"c4 full size: rel-L2 {_rel(got, ref):.3e}")
    assert _rel(got, ref) <= TOL
