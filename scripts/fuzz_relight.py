"""Extended randomised parity sweep of relight_vertices (GEMV, short-row GEMV, tcgen05 split-precision,
CUDA-core tiled paths) against the fp64 oracle: random vertex counts (ragged tiles), faces, band
sizes, batches (1..8, 64, 128, others) and per-row magnitudes 2^U[-40, 40] (the tensor-core path's
row exponents and exact redo).  Not a pytest (minutes of oracle time).
usage: python scripts/fuzz_relight.py [cases] [seed0]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import relight as orelight  # noqa: E402


def main():
    import torch
    import paper_1705_07272_b200 as hs
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 7000
    worst, fails = 0.0, 0
    for case in range(cases):
        rng = np.random.default_rng(seed0 + case)
        faces = int(rng.integers(1, 7))
        k = int(rng.integers(1, 6))
        kf = 4 ** k
        V = int(rng.integers(1, 3000))
        B = int(rng.choice([1, 2, 3, 5, 8, 64, 128, 17, 64]))
        T = synth.transfer_rows(seed0 + case, int(rng.integers(0, 10 ** 6)), V, faces, kf)
        T = (T * np.exp2(rng.integers(-40, 41, size=(V, 1)))).astype(np.float32)
        n = max(k, 2)
        Lp = synth.light_pyramids(seed0 + case, B, faces, n)
        band = np.ascontiguousarray(Lp[:, :, :kf]).astype(np.float32)
        got = hs.relight_vertices(torch.from_numpy(T).cuda(), torch.from_numpy(band).cuda(), faces, kf).cpu().numpy()
        ref = orelight.relight(T.astype(np.float64), band.astype(np.float64), faces, kf)
        # per row, against the row's cancellation-free scale || |T_v| |L|^T || (the fp32 inputs fix the
        # attainable accuracy relative to it; rows of random-sign T can cancel to near zero)
        scale = np.abs(T.astype(np.float64)) @ np.abs(band.reshape(B, -1).astype(np.float64)).T
        err = float(np.max(np.linalg.norm(got - ref, axis=1) / np.maximum(np.linalg.norm(scale, axis=1), 1e-300)))
        worst = max(worst, err)
        if err > 1e-5:
            fails += 1
            print(f"FAIL case {case}: faces {faces} kf {kf} V {V} B {B} worst-row err {err:.3e}")
    print(f"{cases} cases (seeds {seed0}..{seed0 + cases - 1}): {fails} over 1e-5 (per row, relative to the row's "
          f"cancellation-free scale), worst {worst:.3e}")


if __name__ == "__main__":
    main()
