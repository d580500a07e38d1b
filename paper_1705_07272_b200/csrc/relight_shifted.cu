// Fused per-vertex shift + relight:  r_v = < S_{s_v} L , T_v >
// (every pixel/vertex rotates by its own normal angles; the coarser levels
// follow by the recursive h_s / h_t filters; plugged into the light-transport integral).
// DESIGN.md §5.5.
//
// The shifted pyramid of a vertex is never materialised.  The three difference pipelines are
// independent (X -> H, Y -> V, Z -> D), so the work is split into units (face f, field t):
//   prep    : fields_kernel computes the full-resolution difference field F_n (t = X, Y or Z) of
//             every face top-down from its detail coefficients (the shared light L, once per call),
//             stored column-parity split;
//   main    : one CTA holds one unit's field plane (N^2 floats) in shared memory and streams its
//             share of the vertices.  Per vertex: the fused shift + first bottom-up stencil
//             (level n -> n-1) with a register sliding window down each thread's column strip,
//             the [1,1] x [1,2,1] bottom-up to level 0, and the running dot of every shifted
//             detail coefficient of type t with T_v; one partial sum per (vertex, unit);
//   finish  : r_v = sum over units of the partials + sum_f T_v[f][0] L_f[0] (the scaling
//             coefficient is shift invariant).
// Every shift is processed at the finest level (integer shifts have phi = 0), which is exact.
// N = 32, 64 run the unit kernels below; N = 128 precomputes residue planes of the light and
// reads them per vertex instead (csrc/relight_planes.cu), fed by fields_kernel's fp64 fields.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// ------------------------------------------------------------------------------- prep
// fields[f][t][parity][r][c/2] = F_n[r][c] for t in {X, Y, Z}; one CTA per face, top-down over the
// whole (periodic) grid, level by level, ping-ponging through the scratch area.  The recursion
// runs in fp64 and each field value is rounded to fp32 once: fp32 recursion accumulates an
// absolute error ~eps |A| (pixel-value scale, ~1e4 for HDR suns) into every difference.
__global__ void __launch_bounds__(kThreads) fields_kernel(const float* __restrict__ light, int n,
                                                          float* __restrict__ fields, double* __restrict__ scratch) {
  const int f = blockIdx.x;
  const int N = 1 << n;
  const long long NN = (long long)N * N;
  const float* in = light + (long long)f * NN;
  double* buf[2] = {scratch + (long long)f * 6 * NN, scratch + (long long)f * 6 * NN + 3 * NN};
  // level 0 fields are 0; level l+1 from level l
  for (int l = 0; l < n; ++l) {
    const int g = 1 << l, G = 2 * g;
    const double asc = (double)pow2f(l);
    const double* cur = buf[l & 1];
    const bool last = (l + 1 == n);
    double* nxt = buf[(l + 1) & 1];
    for (int idx = threadIdx.x; idx < g * g; idx += blockDim.x) {
      const int i = idx >> l, j = idx & (g - 1);
      double d[2][2][2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int ii = (i + u) & (g - 1), jj = (j + v) & (g - 1);
          const long long o = (long long)ii * g + jj;
          const double H = (double)__ldg(in + (long long)g * g * 1 + o) * asc;
          const double V = (double)__ldg(in + (long long)g * g * 2 + o) * asc;
          const double D = (double)__ldg(in + (long long)g * g * 3 + o) * asc;
          d[u][v][0][0] = H + V + D;
          d[u][v][0][1] = -H + V - D;
          d[u][v][1][0] = H - V - D;
          d[u][v][1][1] = -H - V + D;
        }
      double Xl = 0.0, Yl = 0.0, Zl = 0.0;
      if (l > 0) {
        Xl = __ldcg(cur + idx);
        Yl = __ldcg(cur + g * g + idx);
        Zl = __ldcg(cur + 2 * g * g + idx);
      }
      double cx[2][2], cy[2][2], cz[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        cx[a][0] = d[0][0][a][0] - d[0][0][a][1];
        cx[a][1] = Xl + d[0][0][a][1] - d[0][1][a][0];
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        cy[0][b] = d[0][0][0][b] - d[0][0][1][b];
        cy[1][b] = Yl + d[0][0][1][b] - d[1][0][0][b];
      }
      cz[0][0] = d[0][0][0][0] - d[0][0][0][1] - d[0][0][1][0] + d[0][0][1][1];
      cz[0][1] = d[0][0][0][1] - d[0][0][1][1] - d[0][1][0][0] + d[0][1][1][0];
      cz[1][0] = d[0][0][1][0] - d[0][0][1][1] - d[1][0][0][0] + d[1][0][0][1];
      cz[1][1] = Zl + d[0][0][1][1] - d[0][1][1][0] - d[1][0][0][1] + d[1][1][0][0];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int r = 2 * i + a, c = 2 * j + b;
          {   // natural layout, fp64 (the last level is read by the N = 128 residue planes)
            const int o = r * G + c;
            nxt[o] = cx[a][b];
            nxt[G * G + o] = cy[a][b];
            nxt[2 * G * G + o] = cz[a][b];
          }
          if (last) {
            // final layout: [f][t][parity][r][c/2]
            float* base = fields + (long long)f * 3 * NN;
            const long long o = (long long)(c & 1) * (NN / 2) + (long long)r * (N / 2) + (c >> 1);
            base[o] = (float)cx[a][b];
            base[NN + o] = (float)cy[a][b];
            base[2 * NN + o] = (float)cz[a][b];
          }
        }
    }
    __syncthreads();
    __threadfence_block();
  }
}

// ------------------------------------------------------------------------------- main
constexpr int qpp_pad(int qp, int rows) {   // smallest row length >= qp with rows * q = 16 (mod 32)
  int q = qp;
  while ((rows * q) % 32 != 16) ++q;
  return q;
}

template <int LOG2N>
struct Geo {
  static constexpr int N = 1 << LOG2N;
  static constexpr int G = N / 2;                  // level n-1 side
  // level n-1 columns per thread (N = 128 takes the residue-plane path, csrc/relight_planes.cu)
  static constexpr int CPT = 1;
  static constexpr int TPR = G / CPT;              // threads per level n-1 row
  static constexpr int NS = kThreads / TPR;        // row strips at level n-1
  static constexpr int RS = G / NS;                // output rows per strip
  static constexpr int PADR = 2 * RS + 4;          // wrapped rows appended to the field plane
  // The field is split by column mod SPLIT into SPLIT planes of QP columns: tap k of every thread
  // of a strip is then one plane at consecutive indices (conflict-free).  Rows are padded to QPP
  // so that the two strips sharing a warp (TPR = 16) fall in opposite bank halves.
  static constexpr int SPLIT = 2 * CPT;
  static constexpr int QP = N / SPLIT;
  static constexpr int QPP = TPR >= 32 ? QP : qpp_pad(QP, 2 * RS);
  static constexpr int PLANE = (N + PADR) * QPP;   // one column-class plane, padded
  static constexpr int SCR = 2 * G * G + (G / 2) * (G / 2) + 64;   // one vertex group: S1, S2, red, T block
  static constexpr int smem(int vg) { return (SPLIT * PLANE + vg * SCR) * 4; }
  static_assert(kThreads % TPR == 0 && G % NS == 0 && TPR >= 16, "geometry");
};

// Per-vertex shift classification, once per call (fp64, the same split as the host path).
__global__ void vertex_params_kernel(const float* __restrict__ shifts, long long V, int N, int4* __restrict__ out) {
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= V) return;
  int qy, qx;
  double py, px;
  split_shift((double)shifts[2 * v], N, &qy, &py);
  split_shift((double)shifts[2 * v + 1], N, &qx, &px);
  out[v] = make_int4(qy, qx, __float_as_int((float)py), __float_as_int((float)px));
}

// Named barrier of one vertex group (256 threads; ids 1.. -- id 0 is __syncthreads).
__device__ __forceinline__ void group_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kThreads) : "memory"); }
// One bottom-up level LEV (and, recursively, all coarser ones): shifted fields of level LEV from
// level LEV+1 (periodic), the detail output dotted with T_v's coefficients of type FLD.  Levels
// with more than 64 cells use the whole vertex group (named barrier between levels); the last
// levels (<= 64 cells) run on warp 0 alone (warp-synchronous), the other warps go on.
constexpr int kWarpLevel = 3;
template <int LEV>
struct BU {   // cells per thread of bottom-up level LEV and the offset of its prefetched T values
  static constexpr bool WARP = LEV <= kWarpLevel;
  static constexpr int STRIDE = WARP ? 32 : kThreads;
  static constexpr int CPT = ((1 << (2 * LEV)) + STRIDE - 1) / STRIDE;
  static constexpr int OFF = LEV == 0 ? 0 : BU<(LEV > 0 ? LEV - 1 : 0)>::OFF + BU<(LEV > 0 ? LEV - 1 : 0)>::CPT;
};
template <>
struct BU<0> {
  static constexpr bool WARP = true;
  static constexpr int STRIDE = 32;
  static constexpr int CPT = 1;
  static constexpr int OFF = 0;
};

// T_v's coefficients of type FLD at levels 0 .. TOP that this thread dots, loaded ahead of use
template <int FLD, int LEV, int NT>
__device__ __forceinline__ void prefetch_t(const float* __restrict__ Tv, int tid, float (&tp)[NT]) {
  if constexpr (LEV >= 0) {
    using B = BU<LEV>;
    const float* Tl = Tv + ((long long)(1 + FLD) << (2 * LEV));
#pragma unroll
    for (int k = 0; k < B::CPT; ++k) {
      const int idx = tid + k * B::STRIDE;
      tp[B::OFF + k] = ((!B::WARP || tid < 32) && idx < (1 << (2 * LEV))) ? __ldg(Tl + idx) : 0.f;
    }
    prefetch_t<FLD, LEV - 1, NT>(Tv, tid, tp);
  }
}

template <int LOG2N, int FLD, int LEV, int NT>
__device__ __forceinline__ void bottom_up(const float* src, float* dst, const float (&tp)[NT], int tid, int bar,
                                          float& acc) {
  if constexpr (LEV >= 0) {
    constexpr int g = 1 << LEV, Gs = 2 * g;
    constexpr bool WARP = BU<LEV>::WARP;
    constexpr int STRIDE = BU<LEV>::STRIDE;
    constexpr int CPT = BU<LEV>::CPT;
    const float osc = pow2f(-LEV);
    if (!WARP || tid < 32) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int idx = tid + k * STRIDE;
        if (idx < g * g) {
          const float t = tp[BU<LEV>::OFF + k];
          const int i = idx >> LEV, jj = idx & (g - 1);
          const float* p0 = src + (2 * i) * Gs;
          const float* p1 = p0 + Gs;
          const float* p2 = src + ((2 * i + 2) & (Gs - 1)) * Gs;
          const int c0 = 2 * jj, c1 = 2 * jj + 1, c2 = (2 * jj + 2) & (Gs - 1);
          float fv, dv;
          if (FLD == 0) {
            fv = 0.25f * (p0[c0] + 2.f * p0[c1] + p0[c2] + p1[c0] + 2.f * p1[c1] + p1[c2]);
            dv = 0.25f * (p0[c0] + p1[c0]);
          } else if (FLD == 1) {
            fv = 0.25f * (p0[c0] + 2.f * p1[c0] + p2[c0] + p0[c1] + 2.f * p1[c1] + p2[c1]);
            dv = 0.25f * (p0[c0] + p0[c1]);
          } else {
            fv = 0.25f * ((p0[c0] + 2.f * p0[c1] + p0[c2]) + 2.f * (p1[c0] + 2.f * p1[c1] + p1[c2]) +
                          (p2[c0] + 2.f * p2[c1] + p2[c2]));
            dv = 0.25f * p0[c0];
          }
          if (LEV > 0) dst[idx] = fv;
          acc = fmaf(dv * osc, t, acc);
        }
      }
    }
    if constexpr (LEV > 0) {
      if constexpr (LEV - 1 <= kWarpLevel) {
        if constexpr (WARP) __syncwarp();
        else group_sync(bar);   // level LEV complete before warp 0 reads it
      } else {
        group_sync(bar);
      }
      bottom_up<LOG2N, FLD, LEV - 1, NT>(dst, const_cast<float*>(src), tp, tid, bar, acc);
    }
  }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds(uint32_t a) {
  float x;
  asm("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));   // the plane is read-only after the fill
  return x;
}
__device__ __forceinline__ void mbar_init1(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)));
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_addr(b)),
      "r"(ph)
      : "memory");
}
// one 1D bulk copy global -> shared completing on the group's mbarrier
__device__ __forceinline__ void bulk_to_smem(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(b))
               : "memory");
}

// One (face f, field FLD) unit: vertex group `grp` (256 threads) of the CTA processes vertices
// v0 + grp, v0 + grp + VG, ... < v1.  FLD: 0 = X -> H, 1 = Y -> V, 2 = Z -> D.  The field plane
// (shared by the VG groups) sits in shared memory parity split and padded with PADR wrapped rows,
// so every tap of a thread's strip is an immediate offset from four per-vertex bases; each group
// has its own level n-1 / n-2 scratch and synchronises on its own named barrier.
template <int LOG2N, int FLD, int VG>
__device__ __forceinline__ void unit_body1(const float* plane, float* scratch, uint64_t* mbars, const float* __restrict__ T,
                                          int faces, int f, const int4* __restrict__ vparams, float* __restrict__ partial,
                                          int unit, int units, long long v0, long long v1) {
  using Gm = Geo<LOG2N>;
  constexpr int N = Gm::N, G = Gm::G, RS = Gm::RS, QPP = Gm::QPP, PLANE = Gm::PLANE, SPLIT = Gm::SPLIT;
  constexpr int n = LOG2N;
  constexpr int NTAP = (FLD == 1) ? 3 : 4;
  const int grp = threadIdx.x / kThreads, tid = threadIdx.x % kThreads;
  const int bar = 1 + grp;
  float* S1 = scratch + grp * Gm::SCR;   // shifted field at level n-1 (G x G)
  float* S2 = S1 + G * G;                // level n-2
  float* red = S2 + (G / 2) * (G / 2);
  float* Tb = red + 64;                  // T_v's level n-1 block of type FLD (G x G), bulk-copied
  uint64_t* mb = mbars + grp;
  const long long NN = (long long)N * N;
  const long long Kt = (long long)faces * NN;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int CPT = Gm::CPT;
  const int j = (tid % Gm::TPR) * CPT;  // first level n-1 column owned by this thread
  const int i0 = (tid / Gm::TPR) * RS;  // first output row of this thread's strip
  constexpr int lvl1 = n - 1;
  constexpr uint32_t TB_BYTES = G * G * 4;
  const float qo = 0.25f * pow2f(-lvl1);   // detail scale (power of two: exact)
  auto tblock = [&](long long vv) { return T + vv * Kt + (long long)f * NN + ((long long)(1 + FLD) << (2 * lvl1)); };

  if (tid == 0 && v0 + grp < v1) bulk_to_smem(Tb, tblock(v0 + grp), TB_BYTES, mb);
  uint32_t phase = 0;
  for (long long v = v0 + grp; v < v1; v += VG) {
    const int4 pr = __ldg(vparams + v);
    const float* Tv = T + v * Kt + (long long)f * NN;
    const int qy = pr.x, qx = pr.y;
    const float wy1 = __int_as_float(pr.z), wx1 = __int_as_float(pr.w), wy0 = 1.f - wy1, wx0 = 1.f - wx1;
    float acc = 0.f;
    constexpr int NT = BU<LOG2N - 2>::OFF + BU<LOG2N - 2>::CPT;
    float tp[NT];
    prefetch_t<FLD, LOG2N - 2, NT>(Tv, tid, tp);   // in flight during the fused stencil
    // ---- level n -> n-1: fused shift + first bottom-up, sliding down this thread's rows.
    // window row u = level-n row ((2 i0 - qy - 1) & (N-1)) + u (padded plane, no wrap);
    // column tap k = 0 .. NTK-1 at level n: c = 2j - qx - 1 + k (periodic), in plane c mod SPLIT
    // at index c / SPLIT; output column j + e uses taps 2e .. 2e + NTAP - 1
    constexpr int NTK = 2 * (CPT - 1) + NTAP;
    const int rs = (2 * i0 - qy - 1) & (N - 1);
    uint32_t base[NTK];   // shared-window addresses of the taps at window row 0
#pragma unroll
    for (int k = 0; k < NTK; ++k) {
      const int c = (2 * j - qx + k - 1) & (N - 1);
      base[k] = smem_addr(plane + (c % SPLIT) * PLANE + rs * QPP + c / SPLIT);
    }
    const float ta = wx1, tb0 = wx0 + 2.f * wx1, tb1 = 2.f * wx0 + wx1, tc = wx0;
    const float ua = wy1, ub0 = wy0 + 2.f * wy1, ub1 = 2.f * wy0 + wy1, uc = wy0;
    mbar_wait_parity(mb, phase);   // T_v's level n-1 block has landed
    phase ^= 1;
    // horizontal filters of window row u, streamed: output row r needs rows 2r .. 2r+2 (X) or
    // 2r .. 2r+3 (Y, Z) and is emitted as soon as its last row is filtered
    constexpr int LAST = (FLD == 0) ? 2 : 3;
    {
      float hA[2 * RS + 2], hB[2 * RS + 2];
#pragma unroll
      for (int u = 0; u < 2 * RS + 2; ++u) {
        float x[NTK];
#pragma unroll
        for (int k = 0; k < NTK; ++k) x[k] = lds(base[k] + u * QPP * 4);
        if (FLD == 1) {
          hA[u] = fmaf(wx1, x[0], fmaf(wx0, x[2], x[1]));
          hB[u] = hA[u];
        } else {
          hA[u] = fmaf(ta, x[0], fmaf(tb0, x[1], fmaf(tb1, x[2], tc * x[3 < NTK ? 3 : 0])));
          hB[u] = fmaf(wx1, x[0], wx0 * x[1]);
        }
        if (u >= LAST && ((u - LAST) & 1) == 0) {
          const int r = (u - LAST) >> 1;
          const int w = 2 * r;
          float fl, det;
          if (FLD == 0) {  // X: rows [w1, 1, w0] on taps -1..1, detail rows the same
            fl = 0.25f * fmaf(wy1, hA[w], fmaf(wy0, hA[w + 2], hA[w + 1]));
            det = qo * fmaf(wy1, hB[w], fmaf(wy0, hB[w + 2], hB[w + 1]));
          } else {         // Y, Z: rows tent on taps -1..2; detail rows [w1, w0] on taps -1, 0
            fl = 0.25f * fmaf(ua, hA[w], fmaf(ub0, hA[w + 1], fmaf(ub1, hA[w + 2], uc * hA[w + 3])));
            det = qo * fmaf(wy1, hB[w], wy0 * hB[w + 1]);
          }
          const int o = (i0 + r) * G + j;
          S1[o] = fl;
          acc = fmaf(det, Tb[o], acc);
        }
      }
    }
    group_sync(bar);
    // Tb is free: the next vertex's block streams in during the bottom-up
    if (tid == 0 && v + VG < v1) bulk_to_smem(Tb, tblock(v + VG), TB_BYTES, mb);
    // ---- bottom-up (periodic), ping-pong S1 -> S2 -> S1 ... (compile-time levels)
    bottom_up<LOG2N, FLD, LOG2N - 2, NT>(S1, S2, tp, tid, bar, acc);
    // ---- group reduction of the partial sum (fixed order -> deterministic)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    group_sync(bar);
    if (tid == 0) {
      float sum = 0.f;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) sum += red[w];
      partial[v * units + unit] = sum;
    }
  }
}

template <int LOG2N, int VG>
__global__ void __launch_bounds__(kThreads * VG, 1)
    relight_shifted_unit_kernel(const float* __restrict__ T, long long V, int faces, const float* __restrict__ fields,
                                const int4* __restrict__ vparams, float* __restrict__ partial, int nsplit) {
  using Gm = Geo<LOG2N>;
  constexpr int N = Gm::N, PLANE = Gm::PLANE, SPLIT = Gm::SPLIT, QPP = Gm::QPP;
  extern __shared__ __align__(16) float sm[];
  const int units = 3 * faces;
  const int unit = blockIdx.x % units;
  const int split = blockIdx.x / units;
  const int f = unit / 3, t = unit - 3 * (unit / 3);
  const long long NN = (long long)N * N;
  // field plane -> smem: SPLIT column-class planes [SPLIT][N + PADR][QPP], rows N.. = rows 0..
  // (periodic padding); the prep layout is parity split [2][N][N/2]
  {
    const float* src = fields + ((long long)f * 3 + t) * NN;
    for (int idx = threadIdx.x; idx < SPLIT * PLANE; idx += blockDim.x) {
      const int p = idx / PLANE, rem = idx - p * PLANE;
      const int r = rem / QPP, q = rem - r * QPP;
      if (q < Gm::QP) {
        const int c = q * SPLIT + p;
        sm[idx] = __ldg(src + (long long)(c & 1) * (NN / 2) + (r & (N - 1)) * (N / 2) + (c >> 1));
      }
    }
  }
  __shared__ __align__(8) uint64_t mbars[VG];
  if (threadIdx.x < VG) mbar_init1(&mbars[threadIdx.x]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const long long v0 = V * split / nsplit, v1 = V * (split + 1) / nsplit;
  float* scratch = sm + SPLIT * PLANE;
  if (t == 0) unit_body1<LOG2N, 0, VG>(sm, scratch, mbars, T, faces, f, vparams, partial, unit, units, v0, v1);
  else if (t == 1) unit_body1<LOG2N, 1, VG>(sm, scratch, mbars, T, faces, f, vparams, partial, unit, units, v0, v1);
  else unit_body1<LOG2N, 2, VG>(sm, scratch, mbars, T, faces, f, vparams, partial, unit, units, v0, v1);
}

__global__ void relight_shifted_finish_kernel(const float* __restrict__ partial, const float* __restrict__ T,
                                              const float* __restrict__ light, long long V, int faces, int n,
                                              float* __restrict__ R) {
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int units = 3 * faces;
  const long long NN = 1ll << (2 * n);
  float s = 0.f;
  for (int u = 0; u < units; ++u) s += partial[v * units + u];
  for (int f = 0; f < faces; ++f) s = fmaf(__ldg(T + v * faces * NN + f * NN), __ldg(light + f * NN), s);
  R[v] = s;
}

int num_sms_rs() {
  static int n = 0;
  if (!n) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr int kVG = 3;   // vertex groups per CTA sharing one field plane (1 CTA per SM)

template <int LOG2N, int VG>
hs_status launch_unit_vg(const float* T, long long V, int faces, const float* fields, const int4* shifts,
                         float* partial, cudaStream_t st) {
  constexpr int SM = Geo<LOG2N>::smem(VG);
  static_assert(SM <= 227 * 1024, "shared memory");
  static bool attr = false;
  if (!attr) {
    HS_CHECK_CUDA(cudaFuncSetAttribute(relight_shifted_unit_kernel<LOG2N, VG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, SM),
                  "cudaFuncSetAttribute(relight_shifted_unit_kernel)");
    attr = true;
  }
  const int units = 3 * faces;
  int nsplit = num_sms_rs() / units;   // one CTA per SM
  if (nsplit < 1) nsplit = 1;
  if (nsplit > V) nsplit = (int)V;
  relight_shifted_unit_kernel<LOG2N, VG><<<units * nsplit, kThreads * VG, SM, st>>>(T, V, faces, fields, shifts,
                                                                                    partial, nsplit);
  HS_CHECK_LAUNCH("relight_shifted_unit_kernel");
  return HS_OK;
}

template <int LOG2N>
hs_status launch_unit(const float* T, long long V, int faces, const float* fields, const int4* shifts,
                      float* partial, cudaStream_t st) {
  // three groups: measured 12.5 ms at c4 against 16.5 ms with two (fewer warps to cover the
  // group barriers); four do not fit the N = 128 scratch
  return launch_unit_vg<LOG2N, kVG>(T, V, faces, fields, shifts, partial, st);
}

}  // namespace

bool relight_shifted_fused_supported(int log2n) { return log2n >= 5 && log2n <= 7; }

size_t relight_shifted_fused_workspace_bytes(long long V, int faces, int log2n) {
  const size_t NN = (size_t)1 << (2 * log2n);
  return (size_t)faces * 3 * NN * 4 /*fields*/ + (size_t)faces * 6 * NN * 8 /*fp64 scratch*/ +
         (size_t)V * 3 * faces * 4 /*partials*/ + (size_t)V * 16 /*vertex params*/ + 512 +
         (log2n == 7 ? relight_planes_workspace_bytes(V, faces) + 256 : 0);
}

hs_status launch_relight_shifted_fused(const float* T, long long V, int faces, const float* light, int log2n,
                                       const float* shifts, float* R, void* ws, cudaStream_t st) {
  const size_t NN = (size_t)1 << (2 * log2n);
  float* fields = reinterpret_cast<float*>(ws);
  double* scratch = reinterpret_cast<double*>(fields + (size_t)faces * 3 * NN);
  float* partial = reinterpret_cast<float*>(scratch + (size_t)faces * 6 * NN);
  int4* vp = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(partial + (size_t)V * 3 * faces) + 255) & ~uintptr_t(255));
  fields_kernel<<<faces, kThreads, 0, st>>>(light, log2n, fields, scratch);
  HS_CHECK_LAUNCH("fields_kernel");
  vertex_params_kernel<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(shifts, V, 1 << log2n, vp);
  HS_CHECK_LAUNCH("vertex_params_kernel");
  if (log2n == 7) {   // residue planes (csrc/relight_planes.cu)
    void* pws = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(vp + V) + 255) & ~uintptr_t(255));
    return launch_relight_planes(T, V, faces, light, scratch + 3 * NN, (long long)(6 * NN), vp, R, pws, st);
  }
  hs_status s = HS_OK;
  switch (log2n) {
    case 5: s = launch_unit<5>(T, V, faces, fields, vp, partial, st); break;
    case 6: s = launch_unit<6>(T, V, faces, fields, vp, partial, st); break;
    default: return HS_ERR_UNSUPPORTED;
  }
  if (s != HS_OK) return s;
  relight_shifted_finish_kernel<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(partial, T, light, V, faces, log2n, R);
  HS_CHECK_LAUNCH("relight_shifted_finish_kernel");
  return HS_OK;
}

}  // namespace hs
