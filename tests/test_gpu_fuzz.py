"""Randomised parity sweep of the shift and relight entry points against the fp64 oracle (-m gpu):
seeded random sizes (N = 2 .. 512), face and batch counts, band prefixes and shifts drawn from
every class the path treats differently (zero, multiples of N, dyadic integers, non-dyadic
integers, fractions, negatives, large magnitudes), white-noise or HDR-shaped pyramids."""
import numpy as np
import pytest

import synth
from oracle import relight as orelight
from oracle import shift as oshift

pytestmark = pytest.mark.gpu


def _shift_value(rng, N):
    kind = rng.integers(0, 7)
    if kind == 0:
        return 0.0
    if kind == 1:
        return float(N * rng.integers(-3, 4))
    if kind == 2:                                   # dyadic integer
        return float(rng.integers(-4, 5) * 2 ** rng.integers(0, max(1, int(np.log2(N)))))
    if kind == 3:
        return float(rng.integers(-5 * N, 5 * N))    # any integer
    if kind == 4:
        return float(rng.uniform(-N, N))            # fractional
    if kind == 5:
        return float(rng.integers(0, N) + rng.integers(1, 8) / 8.0)
    return float(rng.uniform(-1e4, 1e4))            # large magnitude


@pytest.mark.parametrize("case", range(64))
def test_shift_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(1000 + case)
    n = int(rng.integers(1, 10))
    N = 1 << n
    faces = int(rng.integers(1, 4 if n >= 8 else 7))
    batch = int(rng.integers(1, 3 if n >= 8 else 5))
    band = int(rng.integers(0, n + 1))
    if rng.random() < 0.5 and n <= 7:
        c = synth.random_signals(case, batch * faces, N * N).reshape(batch, faces, N * N)
    else:
        c = synth.light_pyramids(case, batch, faces, n)
    sh = np.array([[[_shift_value(rng, N), _shift_value(rng, N)] for _ in range(faces)] for _ in range(batch)])
    got = hs.haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(), sh, 2,
                               band).cpu().numpy()
    ref = oshift.shift_coeffs(c, sh, 2, band_levels=band)
    err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert err <= 1e-5, (n, faces, batch, band, err)


@pytest.mark.parametrize("case", range(16))
def test_shift_relight_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(2000 + case)
    n = int(rng.integers(2, 9))
    k = int(rng.integers(1, n + 1))
    faces = int(rng.integers(1, 7))
    B = int(rng.choice([1, 2, 3, 5, 8, 9, 17, 64, 128]))
    V = int(rng.integers(1, 700))
    L = synth.light_pyramids(case, B, faces, n)
    sh = np.array([[[_shift_value(rng, 1 << n), _shift_value(rng, 1 << n)]] * faces for _ in range(B)])
    T = synth.transfer_rows(case, int(rng.integers(0, 10 ** 6)), V, faces, 4 ** k)
    band = hs.haar_shift_coeffs(torch.from_numpy(L).cuda(), sh, 2, k)
    R = hs.relight_vertices(torch.from_numpy(T).cuda(), band, faces, 4 ** k).cpu().numpy()
    ref = orelight.relight(T, oshift.shift_coeffs(L, sh, 2, band_levels=k), faces, 4 ** k)
    err = np.linalg.norm(R - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (n, k, faces, B, V, err)


@pytest.mark.parametrize("case", range(24))
def test_shift_fuzz_white_small(case):
    """White noise with a short band prefix: the worst conditioning (the band holds a tiny share of
    the map's energy, so rounding in the fields is compared against a small result)."""
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(3000 + case)
    n = int(rng.integers(1, 8))
    N = 1 << n
    faces, batch = int(rng.integers(1, 7)), int(rng.integers(1, 5))
    band = int(rng.integers(0, min(n, 2) + 1))
    c = synth.random_signals(case, batch * faces, N * N).reshape(batch, faces, N * N)
    sh = np.array([[[_shift_value(rng, N), _shift_value(rng, N)] for _ in range(faces)] for _ in range(batch)])
    got = hs.haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(), sh, 2,
                               band).cpu().numpy()
    ref = oshift.shift_coeffs(c, sh, 2, band_levels=band)
    err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert err <= 1e-5, (n, faces, batch, band, err)


@pytest.mark.parametrize("case", range(16))
def test_shift1d_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(4000 + case)
    n = int(rng.integers(1, 13))
    N = 1 << n
    faces, batch = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    band = int(rng.integers(0, n + 1))
    c = synth.random_signals(case, batch * faces, N).reshape(batch, faces, N)
    sh = np.array([[[_shift_value(rng, N)] for _ in range(faces)] for _ in range(batch)])
    got = hs.haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(), sh, 1,
                               band).cpu().numpy()
    ref = oshift.shift_coeffs(c, sh, 1, band_levels=band)
    err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert err <= 1e-5, (n, faces, batch, band, err)


@pytest.mark.parametrize("case", range(24))
def test_relight_shifted_fuzz(case):
    """Per-vertex shifts (a7): random N, faces, vertex count (ragged), shift classes."""
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(5000 + case)
    n = int(rng.integers(1, 7))
    N = 1 << n
    faces = int(rng.integers(1, 7))
    V = int(rng.integers(1, 300))
    L = synth.light_pyramids(case, 1, faces, n)[0]
    T = synth.transfer_rows(case, int(rng.integers(0, 10 ** 6)), V, faces, N * N)
    vs = np.array([[_shift_value(rng, N), _shift_value(rng, N)] for _ in range(V)], dtype=np.float32)
    got = hs.relight_vertices_shifted(torch.from_numpy(T).cuda(), torch.from_numpy(L).cuda(),
                                      torch.from_numpy(vs).cuda()).cpu().numpy()
    ref = orelight.relight_shifted(T, L, vs.astype(np.float64))
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (n, faces, V, err)


@pytest.mark.parametrize("case", range(8))
def test_relight_sparse_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(6000 + case)
    n = int(rng.integers(2, 8))
    faces = int(rng.integers(1, 7))
    dense = int(rng.integers(0, min(n - 1, 3) + 1))
    ks = int(faces * 4 ** dense + rng.integers(0, 300))
    V = int(rng.integers(1, 500))
    B = int(rng.choice([1, 2, 5, 16, 64]))
    idx, val = synth.sparse_transfer_rows(case, int(rng.integers(0, 10 ** 6)), V, faces, n, ks, dense)
    L = synth.light_pyramids(case, B, faces, n).reshape(B, -1)
    Ld = torch.from_numpy(L).cuda()
    if case % 2 == 0:                 # per-face layout: the coarse-band cache path
        Ld = Ld.view(B, faces, -1)
    got = hs.relight_vertices_sparse(torch.from_numpy(idx).cuda(), torch.from_numpy(val).cuda(), Ld).cpu().numpy()
    ref = orelight.relight_sparse(idx, val, L)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (n, faces, ks, V, B, err)


@pytest.mark.parametrize("case", range(10))
def test_relight_dense_fuzz(case):
    """Dense relight: GEMV (small batch) and tensor-core (batch % 64 == 0) paths, ragged V, any K."""
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(7000 + case)
    k = int(rng.integers(1, 7))
    faces = int(rng.integers(1, 7))
    B = int(rng.choice([1, 2, 4, 7, 16, 31, 64, 128, 192, 256]))
    V = int(rng.integers(1, 2000))
    T = synth.transfer_rows(case, int(rng.integers(0, 10 ** 6)), V, faces, 4 ** k)
    L = synth.light_pyramids(case, B, faces, k)
    R = hs.relight_vertices(torch.from_numpy(T).cuda(), torch.from_numpy(L).cuda(), faces, 4 ** k).cpu().numpy()
    ref = orelight.relight(T, L, faces, 4 ** k)
    err = np.linalg.norm(R - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (k, faces, B, V, err)


@pytest.mark.parametrize("case", range(16))
def test_relight_triple_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(8000 + case)
    k = int(rng.integers(3, 7))
    kf = 4 ** k
    faces = int(rng.integers(1, 7))
    B = int(rng.choice([1, 3, 8, 64, 128]))
    V = int(rng.integers(1, 400))
    r0 = int(rng.integers(0, 10 ** 6))
    rho = synth.transfer_rows(case, r0, V, faces, kf, synth.STREAM_BRDF)
    vis = synth.transfer_rows(case, r0, V, faces, kf, synth.STREAM_VIS)
    L = synth.light_pyramids(case, B, faces, k)
    rq = hs.haar_pack_qtree(torch.from_numpy(rho).cuda().view(V, faces, kf), k)
    vq = hs.haar_pack_qtree(torch.from_numpy(vis).cuda().view(V, faces, kf), k)
    got = hs.relight_vertices_triple(rq, vq, torch.from_numpy(L).cuda(), faces, kf).cpu().numpy()
    ref = orelight.relight_triple(rho, vis, L, faces, kf)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (k, faces, B, V, err)


@pytest.mark.parametrize("case", range(8))
def test_shift_coarse_fuzz(case):
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(9000 + case)
    n = int(rng.integers(1, 10))
    L0 = int(rng.integers(1, n + 1))
    band = int(rng.integers(0, L0 + 1))
    faces, batch = int(rng.integers(1, 4)), int(rng.integers(1, 3))
    c = synth.light_pyramids(case, batch, faces, n)
    sh = np.array([[[_shift_value(rng, 1 << n), _shift_value(rng, 1 << n)] for _ in range(faces)]
                   for _ in range(batch)])
    got = hs.haar_shift_coeffs_coarse(torch.from_numpy(c).cuda(), sh, L0, band).cpu().numpy()
    for b in range(batch):
        for f in range(faces):
            ref = oshift.shift_coeffs_coarse2d(c[b, f], L0, *sh[b, f])[:4 ** band]
            err = np.linalg.norm(got[b, f] - ref) / max(np.linalg.norm(ref), 1e-30)
            assert err <= 1e-5, (n, L0, band, b, f, err)


@pytest.mark.parametrize("case", range(4))
def test_relight_shifted_fuzz_n128(case):
    """N = 128 (the residue-plane path): random face counts, ragged vertex counts, every shift class
    including exact integers, halves and negatives"""
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(5500 + case)
    n, N = 7, 128
    faces = int(rng.integers(1, 7))
    V = int(rng.integers(1, 40))
    L = synth.light_pyramids(case, 1, faces, n)[0]
    T = synth.transfer_rows(case, int(rng.integers(0, 10 ** 6)), V, faces, N * N)
    vs = np.array([[_shift_value(rng, N), _shift_value(rng, N)] for _ in range(V)], dtype=np.float32)
    got = hs.relight_vertices_shifted(torch.from_numpy(T).cuda(), torch.from_numpy(L).cuda(),
                                      torch.from_numpy(vs).cuda()).cpu().numpy()
    ref = orelight.relight_shifted(T, L, vs.astype(np.float64))
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (faces, V, err)


@pytest.mark.parametrize("B", [1, 3, 64])
def test_relight_dense_long_rows(B):
    """the longest rows the ABI serves in practice: 6 faces x 4^8 = 393216 coefficients per vertex
    (GEMV for small batches, the drained tensor-core chain for 64)"""
    import torch
    import paper_1705_07272_b200 as hs
    k, faces, V = 8, 6, 130
    T = synth.transfer_rows(77, 0, V, faces, 4 ** k)
    L = synth.light_pyramids(78, B, faces, k)
    R = hs.relight_vertices(torch.from_numpy(T).cuda(), torch.from_numpy(L).cuda(), faces, 4 ** k).cpu().numpy()
    ref = orelight.relight(T, L, faces, 4 ** k)
    err = np.linalg.norm(R - ref) / np.linalg.norm(ref)
    print(B, err)
    assert err <= 1e-5, (B, err)


@pytest.mark.parametrize("n,band,sh", [(12, 4, (1234.375, -77.25)), (11, 11, (0.5, 1023.0)), (10, 6, (512.0, 256.0))])
def test_shift_largest_faces(n, band, sh):
    """the largest faces the ABI takes (HS_MAX_LOG2N = 12: 4096^2), white noise, fractional /
    half / dyadic shifts, band or full pyramid"""
    import torch
    import paper_1705_07272_b200 as hs
    N = 1 << n
    c = synth.random_signals(90 + n, 1, N * N).reshape(1, 1, N * N)
    got = hs.haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(),
                               np.array([[list(sh)]]), 2, band).cpu().numpy()
    ref = oshift.shift_coeffs(c, np.array([[list(sh)]]), 2, band_levels=band)
    err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert err <= 1e-5, (n, band, err)


@pytest.mark.parametrize("case", range(3))
def test_relight_shifted_large_faces(case):
    """Per-vertex shifts at N = 256 and 512: the chunked path (a batched shift of the vertex chunk
    with classifications computed on the device, then the row dot) -- the band kernel and the tile
    kernel on device-side FaceParams, every shift class mixed in one chunk."""
    import torch
    import paper_1705_07272_b200 as hs
    rng = np.random.default_rng(9000 + case)
    n = 8 if case < 2 else 9
    N = 1 << n
    faces = 2 if n == 8 else 1
    V = 24
    L = synth.light_pyramids(900 + case, 1, faces, n)[0]
    T = synth.transfer_rows(900 + case, int(rng.integers(0, 10 ** 6)), V, faces, N * N)
    vs = np.array([[_shift_value(rng, N), _shift_value(rng, N)] for _ in range(V)], dtype=np.float32)
    vs[:4] = [[0, 0], [N / 2, 8], [3, 0.5], [64, 128]]
    got = hs.relight_vertices_shifted(torch.from_numpy(T).cuda(), torch.from_numpy(L).cuda(),
                                      torch.from_numpy(vs).cuda()).cpu().numpy()
    ref = orelight.relight_shifted(T, L, vs.astype(np.float64))
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (n, faces, V, err)
