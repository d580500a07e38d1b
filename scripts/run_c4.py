"""Run only relight_vertices_shifted on c4-shaped data (V from argv) -- a short target for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1705_07272_b200 as hs  # noqa: E402

cfg = synth.config("c4")
V = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n, F = cfg.log2n, cfg.faces
T = torch.empty((V, F * 4 ** n), dtype=torch.float32, device="cuda")
hs.hs_fill_transfer(T, 0, F, 4 ** n, cfg.seed, synth.STREAM_T)
L = torch.from_numpy(synth.light_pyramids(cfg.seed, 1, F, n)[0]).cuda()
sv = torch.from_numpy(synth.c4_vertex_shifts(cfg.seed, V, n)).cuda()
R = torch.empty(V, device="cuda")
ws = torch.empty(hs.relight_shifted_workspace_bytes(V, F, n), dtype=torch.uint8, device="cuda")
hs.relight_vertices_shifted(T, L, sv, out=R, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    hs.relight_vertices_shifted(T, L, sv, out=R, workspace=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"c4 fused V={V}: {ms:.3f} ms, {V / ms * 1e3:.3e} vertices/s, {T.numel() * 4 / ms / 1e6:.1f} GB/s")
