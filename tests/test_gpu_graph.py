"""The C ABI is capturable into a CUDA graph (include/haarshift.h): a captured shift + relight step
replays to the same results as direct calls, for a changing light (the graph reads the light buffer
at replay time).  -m gpu."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def test_graph_capture_replays_shift_and_relight():
    import torch
    import paper_1705_07272_b200 as hs
    F, n, kf, V = 6, 6, 1024, 777
    N = 1 << n
    light = torch.from_numpy(synth.light_pyramids(3, 2, F, n)).cuda()
    shifts = np.stack([synth.c3_shifts(n, 360)[[17, 200]]] * F, axis=1)
    T = torch.empty((V, F * kf), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, kf, 4, synth.STREAM_T)
    band = torch.empty((2, F, kf), dtype=torch.float32, device="cuda")
    R = torch.empty((V, 2), dtype=torch.float32, device="cuda")
    ws = torch.empty(hs.haar_shift_workspace_bytes(2, n, F, 2), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):   # warm-up outside capture (attributes, lazy loading)
            hs.haar_shift_coeffs(light, shifts, 2, 5, out=band, workspace=ws)
            hs.relight_vertices(T, band, F, kf, out=R)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        hs.haar_shift_coeffs(light, shifts, 2, 5, out=band, workspace=ws)
        hs.relight_vertices(T, band, F, kf, out=R)
    for seed in (3, 9):
        light.copy_(torch.from_numpy(synth.light_pyramids(seed, 2, F, n)))
        R.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = R.clone()
        ref_band = hs.haar_shift_coeffs(light, shifts, 2, 5)
        ref = hs.relight_vertices(T, ref_band, F, kf)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
