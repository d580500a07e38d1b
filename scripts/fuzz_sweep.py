"""Extended randomised parity sweep of haar_shift_coeffs (2D and 1D) against the fp64 oracle -- the
test_gpu_fuzz generator over many more seeds (not a pytest: minutes of oracle time).
usage: python scripts/fuzz_sweep.py [cases] [seed0]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth  # noqa: E402
from oracle import shift as oshift  # noqa: E402
from test_gpu_fuzz import _shift_value  # noqa: E402


def main():
    import torch
    import paper_1705_07272_b200 as hs
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
    worst, fails = 0.0, 0
    for case in range(cases):
        rng = np.random.default_rng(seed0 + case)
        ndim = 2 if rng.random() < 0.8 else 1
        n = int(rng.integers(1, 10 if ndim == 2 else 13))
        N = 1 << n
        K = N * N if ndim == 2 else N
        faces = int(rng.integers(1, 4))
        batch = int(rng.integers(1, 4))
        band = int(rng.integers(0, n + 1))
        if rng.random() < 0.5:
            c = synth.random_signals(seed0 + case, batch * faces, K).reshape(batch, faces, K)
        elif ndim == 2:
            c = synth.light_pyramids(seed0 + case, batch, faces, n)
        else:
            c = synth.random_signals(seed0 + case, batch * faces, K, "int").reshape(batch, faces, K)
        sh = np.array([[[_shift_value(rng, N) for _ in range(ndim)] for _ in range(faces)] for _ in range(batch)])
        got = hs.haar_shift_coeffs(torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda(), sh, ndim,
                                   band).cpu().numpy()
        ref = oshift.shift_coeffs(c, sh, ndim, band_levels=band)
        err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
        worst = max(worst, err)
        if err > 1e-5:
            fails += 1
            print(f"FAIL case {case}: ndim {ndim} n {n} faces {faces} batch {batch} band {band} err {err:.3e}")
    print(f"{cases} cases (seeds {seed0}..{seed0 + cases - 1}): {fails} over 1e-5, worst rel-L2 {worst:.3e}")


if __name__ == "__main__":
    main()
