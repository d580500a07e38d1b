"""Diagnostic (not a test): split the c5 radiance error against the fp64 oracle into the shift's
and the relight's parts on 20k vertices, and compare the tensor-core relight with an exact fp64
emulation of its fp16 hi/lo split (separates representation from accumulation error)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
import paper_1705_07272_b200 as hs
from oracle import relight as orelight, shift as oshift
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c5")
V, F, n, B, kf = 20000, cfg.faces, cfg.log2n, cfg.frames, cfg.k_face
T = torch.empty((V, F * kf), dtype=torch.float32, device="cuda")
hs.hs_fill_transfer(T, 0, F, kf, cfg.seed, synth.STREAM_T)
light_np = synth.light_pyramids(cfg.seed, B, F, n)
shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
shifted, R = hs.shift_and_relight(torch.from_numpy(light_np).cuda(), shifts, T, F, kf, n)
torch.cuda.synchronize()
rows = np.arange(0, V, 400)
got = R.cpu().numpy()[rows]
Th = T.cpu().numpy()[rows].astype(np.float64)
gband = shifted.cpu().numpy()[:, :, :kf].astype(np.float64)
band = oshift.shift_coeffs(light_np, shifts, 2, band_levels=cfg.band_levels)
ref = Th @ band.reshape(B, -1).T
ref_gb = Th @ gband.reshape(B, -1).T
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print("total", rel(got, ref), "shift part", rel(ref_gb, ref), "relight part", rel(got, ref_gb))
print("band rel err", rel(gband, band), "per-frame max", max(rel(gband[b], band[b]) for b in range(B)))
cond = (np.abs(Th) @ np.abs(band.reshape(B, -1)).T) / np.abs(ref)
print("cond median", np.median(cond), "rms-weighted", np.linalg.norm(np.abs(Th) @ np.abs(band.reshape(B, -1)).T) / np.linalg.norm(ref))
# GEMV-path comparison (fp32 CUDA cores) for the same band
R2 = hs.relight_vertices(T[:V], shifted, F, kf, out=None)
torch.cuda.synchronize()
print("fp32 GEMM path vs fp64 dot of GPU band:", rel(R2.cpu().numpy()[rows], ref_gb))

# emulate the split-precision products exactly in fp64 (no accumulation error)
def split16(x):
    hi = x.astype(np.float16).astype(np.float64)
    lo = ((x - hi) * 2048.0).astype(np.float16).astype(np.float64)
    return hi, lo
Lb = gband.reshape(B, -1).astype(np.float32).astype(np.float64)
mx = np.abs(Lb).max(axis=1)
e = 14 - np.floor(np.log2(mx)).astype(int)
s = np.ldexp(1.0, e)
Ls = (Lb.astype(np.float32) * s[:, None].astype(np.float32)).astype(np.float64)
Lh, Ll = split16(Ls.astype(np.float32))
Th32 = T.cpu().numpy()[rows]
Thh, Thl = split16(Th32)
emu = (Thh @ Lh.T + (Thh @ Ll.T + Thl @ Lh.T) / 2048.0) / s[None, :]
print("tc vs exact-split emulation:", rel(got, emu), " emulation vs fp64 dot:", rel(emu, ref_gb))
