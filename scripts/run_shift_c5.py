"""Run only the c5 shift (64 frames x 6 faces x 256^2) a few times -- a short target for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1705_07272_b200 as hs  # noqa: E402

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c5")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B = cfg.frames
light = torch.from_numpy(synth.light_pyramids(cfg.seed, B, cfg.faces, cfg.log2n)).cuda()
sh = np.broadcast_to(synth.c5_shifts(cfg.seed, B, cfg.log2n)[:, None, :], (B, cfg.faces, 2)).copy()
out = torch.empty_like(light)
ws = torch.empty(hs.haar_shift_workspace_bytes(2, cfg.log2n, cfg.faces, B), dtype=torch.uint8, device="cuda")
for _ in range(2):
    hs.haar_shift_coeffs(light, sh, 2, out=out, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    hs.haar_shift_coeffs(light, sh, 2, out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"shift {cfg.name}: {ms * 1e3:.1f} us/call, {2 * light.numel() * 4 / ms / 1e6:.1f} GB/s")
