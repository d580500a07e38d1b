"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module is the ONLY code both sides of a parity comparison may use. It holds
none of the method's arithmetic: no Haar transform, no shift, no inner product. It only draws
numbers:

* ``splitmix64`` / ``hash_uniform``: a counter-based generator, a pure function of
  (seed, stream, index).  The CUDA fill kernel ``hs_fill_transfer`` (csrc/fill.cu) implements the
  same generator bit for bit, so transfer matrices of tens of GB are generated in place on the GPU
  and any row subset is regenerated here for the oracle.
* ``transfer_rows``: the per-vertex transfer vectors T (BRDF x visibility projected together,
  PAPER.md P:213-222), recipe in DESIGN.md §3.
* ``light_pyramids``: HDR-light-probe-shaped Haar coefficient pyramids (HAAR1 layout, SPEC.md
  S:83), synthesised directly in the coefficient domain (sky gradient + 1 % noise + 3 point "suns"
  per face, PAPER.md P:535 light probes), recipe in DESIGN.md §3.
* shift generators for the BASELINE.json configs c1..c5.

Layouts: a 2D face of side N = 2**n holds N*N unit-square coefficients in HAAR1
order: index 0 is the scaling coefficient, level l (0 <= l < n), type t (H=0, V=1, D=2), cell (i, j)
is at 4**l * (1 + t) + i * 2**l + j.  A 1D signal of length N: index 0 scaling, level l cell k at
2**l + k.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "SEED_BASE", "STREAM_T", "shading_rows", "STREAM_BRDF", "STREAM_VIS", "splitmix64", "hash_u64", "hash_uniform", "level_of_index_2d",
    "level_of_index_1d", "transfer_rows", "light_pyramids", "random_signals", "CONFIGS",
    "Config", "config", "c1_shifts_1d", "c1_shifts_2d", "c3_shifts", "c4_vertex_shifts",
    "c5_shifts", "smooth_sphere_maps", "smooth_sphere_cell_means", "smooth_sphere_eval", "rotation_angles",
]

SEED_BASE = 1705072720          # base seed 1705072720 + config index
STREAM_T = 0x7A11               # counter-hash stream id of the transfer matrix
STREAM_BRDF = 0xB2DF            # triple product (row f3): per-vertex BRDF rows (transfer_rows layout)
STREAM_VIS = 0x7151             # triple product (row f3): per-vertex visibility rows

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output function on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def hash_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """h(seed, stream, idx) = splitmix64(splitmix64(seed + stream * C) + idx), all mod 2**64."""
    with np.errstate(over="ignore"):
        base = splitmix64(np.uint64(seed % 2**64) + np.uint64(stream % 2**64) * _STREAM_MUL)
        return splitmix64(base + np.asarray(idx, dtype=np.uint64))


def hash_uniform(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """u = (h >> 40) / 2**23 - 1 in [-1, 1): 24 random bits, exactly representable in fp32."""
    u24 = (hash_u64(seed, stream, idx) >> np.uint64(40)).astype(np.int64)
    return ((u24 - (1 << 23)).astype(np.float64) / float(1 << 23)).astype(np.float32)


def _floor_log2(k: np.ndarray) -> np.ndarray:
    """floor(log2 k) for integers k >= 1 (exact via frexp); 0 for k = 0."""
    k = np.asarray(k, dtype=np.int64)
    _, e = np.frexp(np.maximum(k, 1).astype(np.float64))
    return (e - 1).astype(np.int64)


def level_of_index_2d(k: np.ndarray) -> np.ndarray:
    """Level l of HAAR1 2D index k (4**l <= k < 4**(l+1)); the scaling index 0 maps to 0."""
    k = np.asarray(k, dtype=np.int64)
    return _floor_log2(k) // 2


def level_of_index_1d(k: np.ndarray) -> np.ndarray:
    return _floor_log2(np.asarray(k, dtype=np.int64))


def transfer_rows(seed: int, row_start: int, row_count: int, faces: int, k_face: int,
                  stream: int = STREAM_T) -> np.ndarray:
    """Rows [row_start, row_start+row_count) of the transfer matrix T, fp32 [rows][faces*k_face].

    T[v][f*k_face + k] = u * 2**-level(k), u = hash_uniform(seed, STREAM_T, v*faces*k_face +
    f*k_face + k); the per-face scaling entry (k = 0) is |u| so radiance has a positive DC part
    (SURVEY.md §8(d) "T values").  Every value is exact in fp32; csrc/fill.cu reproduces it bit
    for bit.
    """
    kt = faces * k_face
    v = np.arange(row_start, row_start + row_count, dtype=np.uint64)[:, None]
    col = np.arange(kt, dtype=np.uint64)[None, :]
    u = hash_uniform(seed, stream, v * np.uint64(kt) + col)
    k = (np.arange(kt) % k_face)
    lev = level_of_index_2d(k)
    scale = np.ldexp(np.float32(1.0), -lev).astype(np.float32)
    t = u * scale[None, :]
    t[:, k == 0] = np.abs(t[:, k == 0])
    return t.astype(np.float32)


def shading_rows(seed: int, row_start: int, row_count: int, faces: int, k_face: int, stream: int) -> np.ndarray:
    """Per-vertex BRDF or visibility rows for the triple product (row f3), fp32 [rows][faces*k_face]:
    transfer_rows(stream) with the details scaled by 1/4 and the scaling entry mapped to
    0.5 + 0.5 |u| -- functions with a positive mean in [0.5, 1) and detail contrast, like a BRDF lobe
    or a visibility mask.  The device side reproduces it bit for bit with
    hs_fill_transfer followed by the same two fp32 operations (bench.py fill_shading)."""
    t = transfer_rows(seed, row_start, row_count, faces, k_face, stream)
    out = (t * np.float32(0.25)).astype(np.float32)
    out[:, ::k_face] = np.float32(0.5) + t[:, ::k_face] * np.float32(0.5)
    return out


STREAM_TS = 0x5A12              # counter-hash stream of the sparse transfer


def sparse_transfer_rows(seed: int, row_start: int, row_count: int, faces: int, log2n: int, k_sparse: int,
                         dense_levels: int = 2):
    """Sparse per-vertex transfer (non-linear approximation):
    K_s (index, value) pairs per vertex over the full pyramids of `faces` faces (index in
    [0, faces * 4**n)).  The first faces * 4**dense_levels entries are every face's coefficients of
    levels < dense_levels (scaling included); the others are hash-drawn detail coefficients with a
    level uniform in [dense_levels, n), a type and a cell.  Values u * 2**-level (|u| for scaling),
    u from hash_uniform.  Returns (idx int32 [rows][K_s], val fp32 [rows][K_s]); csrc/fill.cu's
    hs_fill_sparse_transfer reproduces both bit for bit."""
    N2 = 4 ** log2n
    nd = faces * 4 ** dense_levels
    if k_sparse < nd:
        raise ValueError("k_sparse must cover the dense coarse levels")
    if k_sparse > nd and dense_levels >= log2n:
        raise ValueError("no detail level left to draw the sparse entries from (dense_levels >= log2n)")
    v = np.arange(row_start, row_start + row_count, dtype=np.uint64)[:, None]
    k = np.arange(k_sparse, dtype=np.uint64)[None, :]
    gi = v * np.uint64(k_sparse) + k
    h = hash_u64(seed, STREAM_TS, gi)
    kk = np.broadcast_to(np.arange(k_sparse, dtype=np.int64)[None, :], gi.shape)
    # dense part
    f_d = kk // (4 ** dense_levels)
    c_d = kk % (4 ** dense_levels)
    # hashed part: level, type, cell, face from independent bit fields of h
    nlev = log2n - dense_levels
    lev = dense_levels + ((h >> np.uint64(8)) % np.uint64(max(nlev, 1))).astype(np.int64)
    typ = ((h >> np.uint64(16)) % np.uint64(3)).astype(np.int64)
    face = ((h >> np.uint64(24)) % np.uint64(faces)).astype(np.int64)
    cell = ((h >> np.uint64(32)) & np.uint64(0xFFFFFFFF)).astype(np.int64) % (4 ** lev)
    c_h = (4 ** lev) * (1 + typ) + cell
    dense = kk < nd
    coef = np.where(dense, c_d, c_h)
    fidx = np.where(dense, f_d, face)
    idx = (fidx * N2 + coef).astype(np.int32)
    lvl = np.where(coef == 0, 0, level_of_index_2d(coef))
    u = hash_uniform(seed, STREAM_T, gi)
    val = (u * np.ldexp(np.float32(1.0), -lvl).astype(np.float32)).astype(np.float32)
    val = np.where(coef == 0, np.abs(val), val).astype(np.float32)
    return idx, val


def _sun_params(rng: np.random.Generator, n: int, suns: int):
    N = 1 << n
    r = rng.integers(0, N, size=suns)
    c = rng.integers(0, N, size=suns)
    sigma = rng.uniform(0.7, 2.0, size=suns)
    peak = 10.0 ** rng.uniform(2.0, 4.0, size=suns)
    return r, c, sigma, peak


def light_pyramids(seed: int, batch: int, faces: int, log2n: int, suns: int = 3) -> np.ndarray:
    """HDR-light-probe-shaped HAAR1 pyramids, fp32 [batch][faces][N*N].

    Synthesised directly in the coefficient domain in the averaging convention (detail = signed
    quadrant-mean difference / 4), then scaled to unit-square (x 2**-l) and rounded once to fp32:

    * scaling: 1 + sum over suns of mass / N**2 (sky mean 1 plus the suns' flux);
    * sky gradient 1 + 0.5 cos(pi (r + 1/2) / N): a smooth row-dependent vertical detail
      -0.25 * pi / 2**(l+1) * sin(pi (i + 1/2) / 2**l) at level l;
    * 1 % pixel noise: every detail ~ N(0, (0.01 / 2**(n-l))**2);
    * ``suns`` point suns per face with sigma ~ U[0.7, 2] px and peak ~ 10**U[2, 4]: at level l the
      cell containing the sun gets the details of one bright quadrant of mean min(4 M / W**2, peak)
      (M = 2 pi sigma**2 peak, W = 2**(n-l) pixels per cell side) with the H/V/D sign pattern of
      that quadrant.
    """
    n = log2n
    N = 1 << n
    out = np.empty((batch, faces, N * N), dtype=np.float32)
    for b in range(batch):
        for f in range(faces):
            rng = np.random.default_rng([seed, b, f])
            sr, sc, sig, pk = _sun_params(rng, n, suns)
            mass = 2.0 * math.pi * sig * sig * pk
            c = np.zeros(N * N, dtype=np.float64)
            c[0] = 1.0 + float(mass.sum()) / (N * N)
            for l in range(n):
                g = 1 << l
                W = 1 << (n - l)
                det = rng.normal(0.0, 0.01 / W, size=(3, g, g))
                i = np.arange(g, dtype=np.float64)
                det[1] += (-0.25 * math.pi / (2.0 * g) * np.sin(math.pi * (i + 0.5) / g))[:, None]
                for s in range(suns):
                    ci, cj = sr[s] // W, sc[s] // W
                    a = 1 if (sr[s] % W) >= W // 2 else 0      # row half (0 = top)
                    bq = 1 if (sc[s] % W) >= W // 2 else 0     # column half (0 = left)
                    qmean = min(4.0 * mass[s] / (W * W), pk[s])
                    det[0, ci, cj] += (1.0 if bq == 0 else -1.0) * qmean / 4.0
                    det[1, ci, cj] += (1.0 if a == 0 else -1.0) * qmean / 4.0
                    det[2, ci, cj] += (1.0 if a == bq else -1.0) * qmean / 4.0
                base = 4 ** l
                c[base:4 * base] = (det * (2.0 ** -l)).reshape(-1)
            out[b, f] = c.astype(np.float32)
    return out


def _interval_means(kind: str, p: int, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """Mean of cos(p x) (kind 'c') or sin(p x) (kind 's') over [lo, hi] in closed form."""
    if p == 0:
        return np.full(lo.shape, 1.0 if kind == "c" else 0.0)
    if kind == "c":
        return (np.sin(p * hi) - np.sin(p * lo)) / (p * (hi - lo))
    return (np.cos(p * lo) - np.cos(p * hi)) / (p * (hi - lo))


def _smooth_terms(seed: int, k: int, order: int):
    rng = np.random.default_rng([seed, 0x5F, k])
    terms = [("c", 0, "c", 0, 1.0)]
    for p in range(order + 1):
        for q in range(order + 1):
            if p == 0 and q == 0:
                continue
            amp = 0.35 / (1.0 + p + q)
            for kt in ("c", "s"):
                for kp in ("c", "s"):
                    if (p == 0 and kt == "s") or (q == 0 and kp == "s"):
                        continue
                    terms.append((kt, p, kp, q, float(rng.normal(0.0, amp))))
    return terms


def smooth_sphere_maps(seed: int, count: int, log2n: int, order: int = 3) -> np.ndarray:
    """Smooth lat-long maps (rows theta in [0, pi] top first, columns phi in [0, 2 pi)) as HAAR1
    pyramids, fp32 [count][N*N] -- BRDF-like inputs of the rotation row f1.

    f(theta, phi) = 1 + sum_{p, q <= order} a_pq T_p(theta) S_q(phi), T/S in {cos, sin}, random
    a_pq ~ N(0, (0.35 / (1 + p + q))^2).  Coefficients are exact cell integrals (closed-form means
    of cos / sin over the dyadic intervals), combined per the Haar definition (detail = signed
    quadrant-mean difference / 4, times 2**-l) -- no transform is run."""
    n = log2n
    N = 1 << n
    out = np.empty((count, N * N), dtype=np.float32)
    for kidx in range(count):
        c = np.zeros(N * N, dtype=np.float64)
        for kt, p, kp, q, a in _smooth_terms(seed, kidx, order):
            def means(kind, freq, length, cells):
                e = np.arange(cells + 1, dtype=np.float64) * (length / cells)
                return _interval_means(kind, freq, e[:-1], e[1:])
            c[0] += a * means(kt, p, math.pi, 1)[0] * means(kp, q, 2 * math.pi, 1)[0]
            for l in range(n):
                uc = means(kt, p, math.pi, 2 << l)
                wc = means(kp, q, 2 * math.pi, 2 << l)
                u0, u1, w0, w1 = uc[0::2], uc[1::2], wc[0::2], wc[1::2]
                sc = a * 0.25 * 2.0 ** -l
                base = 4 ** l
                c[base:2 * base] += sc * np.outer(u0 + u1, w0 - w1).reshape(-1)
                c[2 * base:3 * base] += sc * np.outer(u0 - u1, w0 + w1).reshape(-1)
                c[3 * base:4 * base] += sc * np.outer(u0 - u1, w0 - w1).reshape(-1)
        out[kidx] = c.astype(np.float32)
    return out


def smooth_sphere_cell_means(seed: int, count: int, log2n: int, order: int = 3) -> np.ndarray:
    """The finest-level cell means of the same maps, fp64 [count][N][N] (test pin of the above)."""
    N = 1 << log2n
    out = np.zeros((count, N, N))
    e_t = np.arange(N + 1, dtype=np.float64) * (math.pi / N)
    e_p = np.arange(N + 1, dtype=np.float64) * (2 * math.pi / N)
    for kidx in range(count):
        for kt, p, kp, q, a in _smooth_terms(seed, kidx, order):
            out[kidx] += a * np.outer(_interval_means(kt, p, e_t[:-1], e_t[1:]), _interval_means(kp, q, e_p[:-1], e_p[1:]))
    return out


def smooth_sphere_eval(seed: int, k: int, theta, phi, order: int = 3) -> np.ndarray:
    """Point values of map k of smooth_sphere_maps at (theta, phi) (fp64; the analytic ground truth
    of the rotation tests)."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    out = np.zeros(np.broadcast(theta, phi).shape)
    for kt, p, kp, q, a in _smooth_terms(seed, k, order):
        u = np.cos(p * theta) if kt == "c" else np.sin(p * theta)
        w = np.cos(q * phi) if kp == "c" else np.sin(q * phi)
        out += a * u * w
    return out


def rotation_angles(seed: int, count: int) -> np.ndarray:
    """Per-map rotations (alpha = elevation about X, beta = azimuth) in radians, fp64 [count][2]:
    alpha ~ U[-pi/3, pi/3], beta ~ U[0, 2 pi) (row f1)."""
    rng = np.random.default_rng([seed, 0xA7])
    return np.stack([rng.uniform(-math.pi / 3, math.pi / 3, count), rng.uniform(0.0, 2 * math.pi, count)], axis=1)


def random_signals(seed: int, count: int, size: int, kind: str = "normal") -> np.ndarray:
    """Generic seeded fp32 test signals (coefficient vectors or pixel maps)."""
    rng = np.random.default_rng([seed, count, size])
    if kind == "normal":
        return rng.normal(size=(count, size)).astype(np.float32)
    if kind == "int":
        return rng.integers(-8, 9, size=(count, size)).astype(np.float32)
    raise ValueError(kind)


# ---------------------------------------------------------------- shift generators

def c1_shifts_1d(seed: int = SEED_BASE + 1) -> np.ndarray:
    """1D N=8: s in {k/16 : k = -32..160} (incl. 0, 8, negatives) + 64 U(-16, 16) reals."""
    grid = np.arange(-32, 161, dtype=np.float64) / 16.0
    rnd = np.random.default_rng([seed, 1]).uniform(-16.0, 16.0, size=64)
    return np.concatenate([grid, rnd.astype(np.float32).astype(np.float64)])


def c1_shifts_2d(seed: int = SEED_BASE + 1) -> np.ndarray:
    """2D 4x4: (sy, sx) in {k/8 : k = -8..40}^2 (2401 pairs) + 256 random pairs in U(-8, 8)."""
    k = np.arange(-8, 41, dtype=np.float64) / 8.0
    sy, sx = np.meshgrid(k, k, indexing="ij")
    grid = np.stack([sy.ravel(), sx.ravel()], axis=1)
    rnd = np.random.default_rng([seed, 2]).uniform(-8.0, 8.0, size=(256, 2))
    return np.concatenate([grid, rnd.astype(np.float32).astype(np.float64)])


def c3_shifts(log2n: int = 6, frames: int = 360) -> np.ndarray:
    """Per frame f: (0, f N / 360) -- a 1-degree azimuth rotation per frame."""
    N = 1 << log2n
    f = np.arange(frames, dtype=np.float64)
    return np.stack([np.zeros(frames), f * N / 360.0], axis=1)


def c4_vertex_shifts(seed: int, num_vertices: int, log2n: int) -> np.ndarray:
    """Per-vertex local-frame shifts s_v = (theta_N N / pi, phi_N N / (2 pi)), fp32 [V][2], from
    seeded uniform unit normals (rotate by the normal's elevation and azimuth)."""
    N = 1 << log2n
    rng = np.random.default_rng([seed, 4])
    v = rng.normal(size=(num_vertices, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    theta = np.arccos(np.clip(v[:, 1], -1.0, 1.0))              # Y up
    phi = np.mod(np.arctan2(v[:, 0], v[:, 2]), 2.0 * math.pi)
    return np.stack([theta * N / math.pi, phi * N / (2.0 * math.pi)], axis=1).astype(np.float32)


def c5_shifts(seed: int, frames: int, log2n: int) -> np.ndarray:
    """Per frame (sy, sx) ~ U[0, N)^2 stored as fp32 (returned as the exact fp64 of those fp32)."""
    N = 1 << log2n
    s = np.random.default_rng([seed, 5]).uniform(0.0, N, size=(frames, 2)).astype(np.float32)
    return s.astype(np.float64)


# ---------------------------------------------------------------- named configs (BASELINE.json)

@dataclass(frozen=True)
class Config:
    name: str
    log2n: int
    faces: int
    vertices: int
    band_levels: int          # relight uses the per-face prefix 4**band_levels (levels < band_levels)
    frames: int
    seed: int
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def k_face(self) -> int:
        return 4 ** self.band_levels


CONFIGS = {
    "c1": Config("c1", 3, 1, 0, 3, 1, SEED_BASE + 1, "1D N=8 and 2D 4x4, all integer and fractional shifts"),
    "c2": Config("c2", 5, 1, 1000, 5, 1, SEED_BASE + 2, "single 32x32 map, 1 shift, 1k vertices dense T"),
    "c3": Config("c3", 6, 6, 10000, 6, 1, SEED_BASE + 3, "6x64x64 cube map, 10k vertices, per-frame global shift + relight"),
    "c4": Config("c4", 7, 6, 100000, 7, 1, SEED_BASE + 4, "6x128x128 cube map, 100k vertices, per-vertex shifts"),
    "c5": Config("c5", 8, 6, 1000000, 5, 64, SEED_BASE + 5, "6x256x256 cube map, 1M vertices, 64 frames"),
    "c5x": Config("c5x", 8, 6, 1000000, 6, 64, SEED_BASE + 5,
                  "c5 stress variant (SURVEY §8(d)): transfer 6 x 4096 coefficients per vertex (98.3 GB)"),
    "c5s": Config("c5s", 8, 6, 1000000, 8, 64, SEED_BASE + 5,
                  "c5 with sparse top-K transfer (K_s = 256 full-resolution coefficients per vertex, row f2)",
                  {"k_sparse": 256, "dense_levels": 2}),
    "c6r": Config("c6r", 6, 1, 0, 6, 4096, SEED_BASE + 6,
                  "row f1: 4096 lat-long maps of 64 x 64 (BRDF-like, smooth), each rotated by its own (alpha, beta)"),
    "c5t": Config("c5t", 8, 6, 1000000, 5, 64, SEED_BASE + 5,
                  "c5 with the triple product (row f3): per-vertex BRDF and visibility, each 6 x 1024 coefficients"),
    "c7s": Config("c7s", 6, 1, 16384, 5, 64, SEED_BASE + 7,
                  "rows f1 + f3, the paper's shading: 64 frames of a 64 x 64 lat-long HDR light shifted to the "
                  "1024-coefficient band, one smooth BRDF rotated per vertex normal in the Haar domain, "
                  "per-vertex visibility, triple product; 16384 vertices"),
}


def config(name: str) -> Config:
    return CONFIGS[name]
