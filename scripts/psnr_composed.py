"""Accuracy of the composed shading (rows f1 + f3, relight_vertices_brdf_rotated) against the
paper's ground truth (the BRDF rotated in the spatial domain), as PSNR of the
radiance, plus the agreement with the algorithm itself (the chain-rule oracle) as rel-L2.

    python scripts/psnr_composed.py            (on a GPU box; prints one line per size)

Both references are composed from the fp64 oracle only (oracle.rotate.rotate_coeffs = bilinear
resampling at the rotated angles, oracle.rotate.rotate_coeffs_chain = the paper's algorithm,
oracle.relight.relight_triple = the pixel-domain triple integral).  Test infrastructure: reads
oracle/, never the product path's internals.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from oracle import relight as orelight  # noqa: E402
from oracle import rotate as orot  # noqa: E402


def _normals(seed, V):
    v = np.random.default_rng(seed).normal(size=(V, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return np.stack([np.arccos(np.clip(v[:, 1], -1, 1)), np.mod(np.arctan2(v[:, 0], v[:, 2]), 2 * np.pi)], axis=1)


def main():
    import torch
    import paper_1705_07272_b200 as hs
    V, B = 64, 64
    for n, k in ((5, 3), (6, 4), (7, 5)):
        seed = 1800 + n
        brdf = synth.smooth_sphere_maps(seed, 1, n)[0]
        kf = 4 ** k
        vis = synth.shading_rows(seed, 0, V, 1, kf, synth.STREAM_VIS)
        light = synth.light_pyramids(seed, B, 1, n)[:, 0, :]
        nrm = _normals(seed, V)
        dv = torch.from_numpy(np.ascontiguousarray(vis, dtype=np.float32)).cuda()
        vq = hs.haar_pack_qtree(dv.view(V, 1, kf), k).view(V, kf)
        got = hs.relight_vertices_brdf_rotated(torch.from_numpy(brdf).cuda(), nrm, vq,
                                               torch.from_numpy(np.ascontiguousarray(light)).cuda(), k)
        torch.cuda.synchronize()
        got = got.cpu().numpy().astype(np.float64)

        def ref(rotate):
            rho = np.stack([rotate(brdf.astype(np.float64), float(nrm[v, 0]), float(nrm[v, 1]))[:kf]
                            for v in range(V)])
            return orelight.relight_triple(rho, vis.astype(np.float64), light[:, None, :].astype(np.float64), 1, kf)

        spatial, chain = ref(orot.rotate_coeffs), ref(orot.rotate_coeffs_chain)
        rmse = float(np.sqrt(np.mean((got - spatial) ** 2)))
        psnr = 20 * np.log10(float(np.abs(spatial).max()) / rmse)
        rmse_a = float(np.sqrt(np.mean((chain - spatial) ** 2)))
        psnr_a = 20 * np.log10(float(np.abs(spatial).max()) / rmse_a)
        rel = float(np.linalg.norm(got - chain) / np.linalg.norm(chain))
        print(f"N={2 ** n:4d} band 4^{k}: radiance PSNR vs spatial rotation {psnr:6.2f} dB "
              f"(the algorithm's own, fp64 oracle: {psnr_a:6.2f} dB); GPU vs chain oracle rel-L2 {rel:.2e}")


if __name__ == "__main__":
    main()
