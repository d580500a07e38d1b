"""Sharding is exact (-m gpu): every relight entry point, called on a block of
vertex rows, returns BITWISE the same rows as the unsharded call -- the multi-GPU path splits the
vertex rows into contiguous blocks per rank (paper_1705_07272_b200.dist.shard_rows), so this is
what makes the gathered radiance of N ranks equal the 1-GPU radiance.  The split offsets are
deliberately not multiples of the 128-row tensor-core tile (nor of the GEMV's row groups), and
the blocks are those shard_rows gives for 3 and 7 ranks plus a few ragged cuts.  One GPU runs every
block in turn (no kernel waits on another)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _blocks(V):
    from paper_1705_07272_b200 import dist as hsdist
    cuts = [[hsdist.shard_rows(V, w, r) for r in range(w)] for w in (3, 7)]
    ragged = [(0, 1), (1, 130), (131, 255), (386, V - 386)]
    return cuts + [ragged]


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


@pytest.mark.parametrize("B", [1, 3, 8, 13, 64, 128])
def test_relight_vertices_shards_bitwise(B):
    import torch
    import paper_1705_07272_b200 as hs
    F, kf, V = 6, 1024, 1000
    T = torch.empty((V, F * kf), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, kf, synth.SEED_BASE + 11, synth.STREAM_T)
    L = _dev(synth.light_pyramids(80, B, F, 5))
    full = hs.relight_vertices(T, L, F, kf)
    for blocks in _blocks(V):
        got = torch.empty_like(full)
        for s, n in blocks:
            hs.relight_vertices(T[s:s + n], L, F, kf, out=got[s:s + n])
        torch.cuda.synchronize()
        assert torch.equal(got, full), (B, blocks)


@pytest.mark.parametrize("B", [64, 5])
def test_relight_triple_shards_bitwise(B):
    import torch
    import paper_1705_07272_b200 as hs
    F, k, V = 6, 5, 700
    kf = 4 ** k
    rq = hs.haar_pack_qtree(_dev(synth.shading_rows(81, 0, V, F, kf, synth.STREAM_BRDF)).view(V, F, kf), k)
    vq = hs.haar_pack_qtree(_dev(synth.shading_rows(81, 0, V, F, kf, synth.STREAM_VIS)).view(V, F, kf), k)
    L = _dev(synth.light_pyramids(82, B, F, k))
    full = hs.relight_vertices_triple(rq, vq, L, F, kf)
    for blocks in _blocks(V):
        got = torch.empty_like(full)
        for s, n in blocks:
            hs.relight_vertices_triple(rq[s:s + n], vq[s:s + n], L, F, kf, out=got[s:s + n])
        torch.cuda.synchronize()
        assert torch.equal(got, full), (B, blocks)


@pytest.mark.parametrize("B", [64, 3])
def test_relight_sparse_shards_bitwise(B):
    import torch
    import paper_1705_07272_b200 as hs
    F, n, ks, V = 6, 6, 64, 900
    idx = torch.empty((V, ks), dtype=torch.int32, device="cuda")
    val = torch.empty((V, ks), dtype=torch.float32, device="cuda")
    hs.hs_fill_sparse_transfer(idx, val, 0, F, n, 1, 83)
    L = _dev(synth.light_pyramids(84, B, F, n))
    full = hs.relight_vertices_sparse(idx, val, L)
    for blocks in _blocks(V):
        got = torch.empty_like(full)
        for s, c in blocks:
            hs.relight_vertices_sparse(idx[s:s + c], val[s:s + c], L, out=got[s:s + c])
        torch.cuda.synchronize()
        assert torch.equal(got, full), (B, blocks)


@pytest.mark.parametrize("n", [5, 7])
def test_relight_shifted_shards_bitwise(n):
    import torch
    import paper_1705_07272_b200 as hs
    F, V = 6, 600
    T = torch.empty((V, F * 4 ** n), dtype=torch.float32, device="cuda")
    hs.hs_fill_transfer(T, 0, F, 4 ** n, synth.SEED_BASE + 12, synth.STREAM_T)
    L = _dev(synth.light_pyramids(85, 1, F, n)[0])
    sv = _dev(synth.c4_vertex_shifts(86, V, n))
    full = hs.relight_vertices_shifted(T, L, sv)
    for blocks in _blocks(V):
        got = torch.empty_like(full)
        for s, c in blocks:
            hs.relight_vertices_shifted(T[s:s + c], L, sv[s:s + c], out=got[s:s + c])
        torch.cuda.synchronize()
        assert torch.equal(got, full), (n, blocks)
