"""Run only the 1D Haar-domain shift (shift1d_kernel): 4096 signals of N = 4096, fractional shifts --
a short target for ncu (config c1 is the tiny parity case)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1705_07272_b200 as hs  # noqa: E402

n, S = 12, 4096
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x = torch.from_numpy(synth.random_signals(synth.SEED_BASE + 11, S, 1 << n)).cuda().view(S, 1, 1 << n)
sh = np.random.default_rng(11).uniform(0, 1 << n, size=(S, 1, 1))
out = torch.empty_like(x)
hs.haar_shift_coeffs(x, sh, 1, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    hs.haar_shift_coeffs(x, sh, 1, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"shift1d {S} x N={1 << n}: {ms * 1e3:.1f} us/call, {2 * x.numel() * 4 / ms / 1e6:.1f} GB/s")
