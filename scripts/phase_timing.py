"""Debug: per-phase clock64 profile of the 2D shift tile kernel (needs lib/libhaarshift_dbg.so built
with -DHS_PHASE_TIMING).  Not part of the product or tests."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1705_07272_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_1705_07272_b200", "lib", "libhaarshift_dbg.so")
lib = _lib.load()
lib.hs_debug_phase_dump.restype = ctypes.c_int
lib.hs_debug_phase_dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
import paper_1705_07272_b200 as hs  # noqa: E402

cfg = synth.config("c5")
B = cfg.frames
light = torch.from_numpy(synth.light_pyramids(cfg.seed, B, cfg.faces, cfg.log2n)).cuda()
sh = np.broadcast_to(synth.c5_shifts(cfg.seed, B, cfg.log2n)[:, None, :], (B, cfg.faces, 2)).copy()
out = torch.empty_like(light)
for _ in range(3):
    hs.haar_shift_coeffs(light, sh, 2, out=out)
torch.cuda.synchronize()
ntile = 16 * B * cfg.faces
buf = np.zeros(ntile * 16, dtype=np.int64)
assert lib.hs_debug_phase_dump(buf.ctypes.data, buf.size) == 0
ph = buf.reshape(ntile, 16)[:, :10].astype(np.float64)
names = ["start", "window starts", "loads issued + group A wait", "(marker)", "level c+1 fields + group B wait",
         "level m-1 fields", "field X: children + fused", "fields Y, Z: children + fused", "bottom-up", "publish"]
d = np.diff(ph, axis=1)
tot = ph[:, 9] - ph[:, 0]
print(f"CTA lifetime (phase 0 -> 9): median {np.median(tot):.0f} cycles, mean {tot.mean():.0f}")
for i in range(9):
    print(f"{names[i + 1]:>20s}: median {np.median(d[:, i]):8.0f}  mean {d[:, i].mean():8.0f} cycles")
