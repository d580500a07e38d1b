// 2D Haar-domain shift, register-streaming form for working levels m = 6, 7, 8 (SURVEY.md §8(a)
// rows a2-a4).  Same arithmetic as shift2d.cu's tile kernel -- the exact
// difference-domain top-down from the detail coefficients (P:331, P:408, P:463 made exact), the
// shift of the level-m fields fused with the first bottom-up step (eq:pde1-2 P:416-425, P:459,
// P:508), and the paper's [1,1] (x) [1,2,1] / 4 bottom-up (eq:conv/tker/sker P:466-497) --
// organised so that no field ever goes through shared memory:
//
//   * one CTA per (face, band of HB output rows at level m-1), one WARP per field F in {X, Y, Z};
//     the three fields are independent through the whole recursion (X_{l+1} needs X_l and the
//     details only, X'_l needs X'_{l+1} only), so each warp carries one field's state;
//   * at CTA start the CTA stages every DETAIL row the band needs at levels m-1, m-2, c = m-3
//     (cp.async of the fp32 values; columns rotated by the face's window offset and interleaved so
//     that a lane's window element is one conflict-free shared load at an immediate offset) and
//     the unshifted level-c field rows coarse_fields_kernel left in the workspace into shared
//     memory (<= 53 KB, four CTAs per SM): the three field warps share one read of the pyramid;
//   * LPR = 2^(m-3) lanes cover a full row at level m-1 with CPL = 4 output columns per lane (a
//     warp holds 32 / LPR row groups, each streaming its own RB-row band); the lane's window at
//     every level is the set of columns its outputs depend on, in SHIFTED coordinates (the column
//     shift Qx is uniform per face); the column parities are folded into zero-padded tap vectors;
//   * the warp walks its band top to bottom, one PARENT row p at level m-1 per step: the parent's
//     field row (two at a time from the level m-2 row p/2, itself from the level-c fields), its two
//     level-m child rows, their horizontal shift stencils, the vertical stencil -- the child rows
//     of one parent feed up to three output rows, with per-face weights that absorb the parity of
//     Qy -- and the bottom-up m-1 -> m-2 -> c in registers (the [1,2,1] neighbour column is a
//     shuffle from the next lane);
//   * outputs at levels m-1, m-2, c go straight to global memory (float4 / float2 / float rows);
//     the shifted level-c fields go to the workspace for coarse_finish_kernel (levels < c).
//
// Fields are fp64 throughout (DESIGN.md §4.1 error model); a detail row is widened to fp64 (in
// averaging units) once per lane when its window is loaded.  Band halos: the X field's bottom-up is [1,1] vertically (no halo); Y and Z use [1,2,1]
// and compute 3 extra rows at level m-1 (and 1 at level m-2) below the band.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

constexpr int CPL = 4;                   // level m-1 output columns per lane
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double p2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// Children at the next finer level of one field, window-relative: child t (t < NCH) sits under
// parent index u = t >> 1 with column parity b = t & 1; row parity A.  F: parent field row, Dp / Dq:
// the parent row's details and the next row's (H, V, D in averaging units, i.e. already scaled by
// 2^level).  The formulas are shift2d.cu's top-down written per field (q1: column q+1, p1: row p+1):
//   X: (A,0) 2(H +- D)          (A,1) X + (-H+V-D) - (H+V+D)[q1]  |  X + (-H-V+D) - (H-V-D)[q1]
//   Y: (0,b) 2(V +- D)          (1,b) Y + d_1b - d_0b[p1]
//   Z: (0,0) 4D   (0,1) 2(V-D - (V+D)[q1])   (1,0) 2(H-D - (H+D)[p1])
//      (1,1) Z + d11 - d10[q1] - d01[p1] + d00[p1,q1]
template <int FLD, int A, int NCH, int WF, int WD>
__device__ __forceinline__ void children(const double (&F)[WF], const double (&Dp)[3][WD], const double (&Dq)[3][WD],
                                         double (&out)[NCH]) {
#pragma unroll
  for (int t = 0; t < NCH; ++t) {
    const int u = t >> 1, b = t & 1;
    const double H = Dp[0][u], V = Dp[1][u], D = Dp[2][u];
    double r;
    if (FLD == 0) {
      if (b == 0) {
        r = 2.0 * (A == 0 ? H + D : H - D);
      } else {
        const double H1 = Dp[0][u + 1], V1 = Dp[1][u + 1], D1 = Dp[2][u + 1];
        r = F[u] + (A == 0 ? (-H + V - D) - (H1 + V1 + D1) : (-H - V + D) - (H1 - V1 - D1));
      }
    } else if (FLD == 1) {
      if (A == 0) {
        r = 2.0 * (b == 0 ? V + D : V - D);
      } else {
        const double H2 = Dq[0][u], V2 = Dq[1][u], D2 = Dq[2][u];
        r = F[u] + (b == 0 ? (H - V - D) - (H2 + V2 + D2) : (-H - V + D) + (H2 - V2 + D2));
      }
    } else {
      if (A == 0 && b == 0) {
        r = 4.0 * D;
      } else if (A == 0) {
        const double V1 = Dp[1][u + 1], D1 = Dp[2][u + 1];
        r = 2.0 * ((V - D) - (V1 + D1));
      } else if (b == 0) {
        const double H2 = Dq[0][u], D2 = Dq[2][u];
        r = 2.0 * ((H - D) - (H2 + D2));
      } else {
        const double H1 = Dp[0][u + 1], V1 = Dp[1][u + 1], D1 = Dp[2][u + 1];
        const double H2 = Dq[0][u], V2 = Dq[1][u], D2 = Dq[2][u];
        const double H3 = Dq[0][u + 1], V3 = Dq[1][u + 1], D3 = Dq[2][u + 1];
        r = F[u] + (((-H - V + D) + (-H1 + V1 + D1)) + ((H2 - V2 + D2) + (H3 + V3 + D3)));
      }
    }
    out[t] = r;
  }
}

template <int N>
__device__ __forceinline__ void realign(bool sh, const double* src, double (&dst)[N]) {   // dst[i] = src[i + sh]
#pragma unroll
  for (int i = 0; i < N; ++i) dst[i] = sh ? src[i + 1] : src[i];
}

// Band geometry of one face.  LPR lanes hold a level m-1 row (CPL columns each); a warp holds GPW
// row groups; a row group streams RB output rows; a CTA (3 field warps) covers HB = GPW * RB rows.
// Band geometry of one face at working level M.  LPR lanes hold a level M-1 row (CPL columns each);
// a warp holds GPW row groups; a row group streams RB output rows; a CTA (3 field warps) covers
// HB = GPW * RB rows.  Shared memory holds, per level, the staged rows with the columns rotated by
// the face's window offset and interleaved (column c' -> (c' % PER) * (LPR + PAD) + c' / PER), so
// that lane Lg's window element u is at Lg + a compile-time offset -- bank-conflict free -- and the
// detail values are fp32 (widened to fp64 in averaging units when a lane loads its window).
template <int M>
struct SG {
  static constexpr int LPR = 1 << (M - 3), GPW = 32 / LPR;
  static constexpr int H1 = 1 << (M - 1), H2 = H1 >> 1, HC = H1 >> 2;
  static constexpr int RB = (H1 / GPW) < 16 ? (H1 / GPW) : 16;
  static constexpr int HB = GPW * RB, NBANDS = H1 / HB;
  static constexpr int ROW1 = 4 * (LPR + 1), ROW2 = 2 * (LPR + 1), ROW3 = LPR + 2, ROWW = LPR + 1;
  static constexpr int mn(int a, int b) { return a < b ? a : b; }
  static constexpr int NR1 = mn(HB + 6, H1), NR2 = mn((HB + 6) / 2 + 2, H2), NR3 = mn((HB + 6) / 4 + 2, HC),
                       NRW = mn((HB + 6) / 4 + 1, HC);
  static constexpr int PLANE1 = NR1 * ROW1, PLANE2 = NR2 * ROW2, PLANE3 = NR3 * ROW3, PLANEW = NRW * ROWW;
  static constexpr int r4(int x) { return (x + 3) & ~3; }
  static constexpr int OFF2 = r4(3 * PLANE1), OFF3 = r4(OFF2 + 3 * PLANE2), NDET = r4(OFF3 + 3 * PLANE3);   // doubles
  static constexpr int OFFW = NDET / 2;           // in doubles, after the NDET floats
  static constexpr int SMEM = NDET * 4 + 3 * PLANEW * 8;
};
constexpr int kStreamMaxBands = SG<8>::NBANDS;
constexpr int kStreamThreads = 96;             // warps X, Y, Z
constexpr int kStreamSmem = SG<8>::SMEM > SG<7>::SMEM ? (SG<8>::SMEM > SG<6>::SMEM ? SG<8>::SMEM : SG<6>::SMEM)
                                                      : (SG<7>::SMEM > SG<6>::SMEM ? SG<7>::SMEM : SG<6>::SMEM);
static_assert(kStreamSmem <= 56 * 1024, "four CTAs per SM");

// Rows [base, base + n) modulo H of one level staged in shared memory.
struct RowSet {
  int base, n, H;
  __device__ int row(int r) const { return (r - base) & (H - 1); }
};
__device__ __forceinline__ RowSet make_rows(int first, int last, int H, int cap) {   // rows first .. last
  RowSet rs;
  rs.base = first;
  rs.n = last - first + 1;
  if (rs.n > H) rs.n = H;
  if (rs.n > cap) rs.n = cap;   // unreachable: cap is the static maximum of n
  rs.H = H;
  return rs;
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
// Stage 3 planes of rows rs of one level (plane stride pstride in global) at element offsets
// t * PLANE + j * ROW + pos of sf (see SG): position pos = k (LPR + PADR) + q holds rotated column
// c' = PER q + k (q = LPR .. LPR + PADR - 1 repeat q = 0 ..), source column (c' + s) mod H.  One
// warp per row, the lanes over the positions (each lane's source columns are row-independent).
template <int PER, int LPR, int PADR, int ROW, int PLANE, typename T>
__device__ __forceinline__ void stage_rows(const T* __restrict__ g0, long long pstride, const RowSet& rs, int s,
                                           T* __restrict__ sf) {
  constexpr int SUB = LPR + PADR, NI = (ROW + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hm = rs.H - 1;
  int col[NI];   // source column of each of the lane's positions: the same for every row
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int pos = lane + 32 * i;
    const int k = pos / SUB, q = pos - k * SUB;
    col[i] = (PER * (q >= LPR ? q - LPR : q) + k + s) & hm;
  }
  const int nrow = 3 * rs.n;
  for (int row = warp; row < nrow; row += kStreamThreads / 32) {
    const int t = (row >= rs.n) + (row >= 2 * rs.n), j = row - t * rs.n;
    const T* src = g0 + (long long)t * pstride + (long long)((rs.base + j) & hm) * rs.H;
    T* dst = sf + t * PLANE + j * ROW + lane;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (lane + 32 * i < ROW) {
        if constexpr (sizeof(T) == 4) cp_async4(dst + 32 * i, src + col[i]); else cp_async8(dst + 32 * i, src + col[i]);
      }
    }
  }
}

template <int M, int FLD>
__device__ __forceinline__ void stream_task(const ShiftArgs& args, const FaceParam& P, int g, int J0,
                                            const float* S, const double* SW, const RowSet& R1, const RowSet& R2,
                                            const RowSet& R3, const RowSet& RW) {
  using G = SG<M>;
  constexpr int NCE = (FLD == 1) ? 2 * CPL + 2 : 2 * CPL + 3;  // level-M children from the even start 2 P1
  constexpr int NT = (FLD == 1) ? 4 : 5;                       // horizontal taps incl. the parity pad
  constexpr int W1F = CPL + 1;                                 // level M-1 fields (window at P1)
  constexpr int W1E = W1F + 1;                                 // computed from the even start P1 - p1odd
  constexpr int W1D = (FLD == 1) ? CPL + 1 : CPL + 2;          // level M-1 detail columns
  constexpr int W2F = 3, W2D = (FLD == 1) ? 3 : 4;             // level M-2 (aligned at P2)
  constexpr int W3F = 2, W3D = (FLD == 1) ? 2 : 3;             // level c
  constexpr int LPR = G::LPR, H1 = G::H1, H2 = G::H2, HC = G::HC, RB = G::RB, C = M - 3;

  const int lane = threadIdx.x & 31;
  const int Lg = lane & (LPR - 1), grp = lane / LPR;
  const int I0 = J0 + grp * RB;

  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  const int oband = args.band;
  double* wsS = reinterpret_cast<double*>(reinterpret_cast<char*>(args.ws) + (long long)g * args.ws_face_stride);
  const float* S1 = S + Lg;
  const float* S2 = S + G::OFF2 + Lg;
  const float* S3 = S + G::OFF3 + Lg;
  const double* SWl = SW + FLD * G::PLANEW + Lg;
  // unit-square -> averaging: x 2^level, exact in fp32 before the widening (|detail| < 2^120)
  constexpr float asc1 = float(1u << (M - 1)), asc2 = float(1u << (M - 2)), asc3 = float(1u << C);

  // column parities of the windows (level M children start 2 P1, c0 = 2 P1 + codd; P1 = 4 Lg + s1,
  // P2 = P1 >> 1 = 2 Lg + s2, P3 = P2 >> 1 = Lg + s3): the staged rows are rotated by s1, s2, s3
  const int cq = -P.Qx - 1;
  const bool codd = (cq & 1) != 0, p1odd = ((cq >> 1) & 1) != 0;
  const bool sel2 = ((cq >> 2) & 1) != 0;
  const int R0 = 2 * I0 - P.Qy - 1;
  const int o = R0 & 1;
  const int pbase = R0 >> 1;
  const int qh = (P.Qy + 1) >> 1;

  // weights: w1 = phi, w0 = 1 - phi.  Horizontal taps, zero-padded for the column parity codd:
  // X, Z: B = [w1, w0 + 2 w1, 2 w0 + w1, w0] (field) and [w1, w0] (detail); Y: A = [w1, 1, w0].
  const double wy1 = (double)P.wy, wy0 = 1.0 - wy1, wx1 = (double)P.wx, wx0 = 1.0 - wx1;
  double TA[NT], TB[3];
  {
    double base[NT];
    if (FLD == 1) {
      base[0] = wx1; base[1] = 1.0; base[2] = wx0; base[3] = 0.0;
    } else {
      base[0] = wx1; base[1] = wx0 + 2.0 * wx1; base[2] = 2.0 * wx0 + wx1; base[3] = wx0; base[4] = 0.0;
    }
#pragma unroll
    for (int v = 0; v < NT; ++v) TA[v] = codd ? (v ? base[v - 1] : 0.0) : base[v];
    TB[0] = codd ? 0.0 : wx1;
    TB[1] = codd ? wx1 : wx0;
    TB[2] = codd ? wx0 : 0.0;
  }
  // Vertical: output row i reads level-M rows R0(i) = 2i - Qy - 1 .. +2 (X, taps A = [w1, 1, w0])
  // or .. +3 (Y, Z, taps B).  Parent p's rows 2p (even) and 2p + 1 (odd) complete one output row
  // ("done") and seed the next ones (carries c1, c2); the split of the taps between them depends on
  // o = R0 & 1 only, so it is a set of per-face weights (a* -> done, b* -> c1, g* -> c2).
  // V^' / D^' use the 2 taps [w1, w0] on rows R0, R0 + 1 (v* -> done, vg -> carry).
  const double by0 = wy1, by1 = wy0 + 2.0 * wy1, by2 = 2.0 * wy0 + wy1, by3 = wy0;
  double ae, ao, be, bo, ge, go, ve, vo, vg;
  if (FLD == 0) {
    ae = o ? 1.0 : wy0; be = o ? 0.0 : wy1; ao = o ? wy0 : 0.0; bo = o ? wy1 : 1.0;
    ge = go = ve = vo = vg = 0.0;
  } else {
    ae = o ? by3 : by2; ao = o ? 0.0 : by3; be = o ? by1 : by0; bo = o ? by2 : by1; ge = 0.0; go = o ? by0 : 0.0;
    ve = o ? wy0 : wy1; vo = o ? 0.0 : wy0; vg = o ? wy1 : 0.0;
  }

  // ---------------------------------------------------------------- windows (shared memory, fp64)
  auto window1 = [&](int p, double (&D)[3][W1D]) {
    const float* r = S1 + R1.row(p) * G::ROW1;
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < W1D; ++u) D[t][u] = (double)(r[t * G::PLANE1 + (u & 3) * (LPR + 1) + (u >> 2)] * asc1);
  };
  auto window2 = [&](int p2, double (&D)[3][W2D]) {
    const float* r = S2 + R2.row(p2) * G::ROW2;
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < W2D; ++u) D[t][u] = (double)(r[t * G::PLANE2 + (u & 1) * (LPR + 1) + (u >> 1)] * asc2);
  };
  auto window3 = [&](int p3, double (&D)[3][W3D]) {
    const float* r = S3 + R3.row(p3) * G::ROW3;
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < W3D; ++u) D[t][u] = (double)(r[t * G::PLANE3 + u] * asc3);
  };

  // ---------------------------------------------------------------- level M-1 fields, two rows at a time
  int cur_g = -(1 << 30);
  double F1g[2 * W1F];
  auto group1 = [&](int g2) {   // level M-1 field rows 2 g2, 2 g2 + 1 (level M-2 row g2)
    cur_g = g2;
    const int p3 = g2 >> 1;
    double F3[W3F];
    {
      const double* wrow = SWl + RW.row(p3) * G::ROWW;
#pragma unroll
      for (int v = 0; v < W3F; ++v) F3[v] = wrow[v];
    }
    double F2e[4], F2[W2F];
    {
      double D3a[3][W3D];
      window3(p3, D3a);
      if (g2 & 1) {
        double D3b[3][W3D];
        if (FLD != 0) window3(p3 + 1, D3b);
        children<FLD, 1, 4>(F3, D3a, D3b, F2e);
      } else {
        children<FLD, 0, 4>(F3, D3a, D3a, F2e);
      }
    }
    realign<W2F>(sel2, F2e, F2);
    double D2a[3][W2D], D2b[3][W2D];
    window2(g2, D2a);
    if (FLD != 0) window2(g2 + 1, D2b);
    double F1e[W1E], F1r[W1F];
    children<FLD, 0, W1E>(F2, D2a, D2a, F1e);
    realign<W1F>(p1odd, F1e, F1r);
#pragma unroll
    for (int u = 0; u < W1F; ++u) F1g[u] = F1r[u];
    children<FLD, 1, W1E>(F2, D2a, D2b, F1e);
    realign<W1F>(p1odd, F1e, F1r);
#pragma unroll
    for (int u = 0; u < W1F; ++u) F1g[W1F + u] = F1r[u];
  };

  // ---------------------------------------------------------------- bottom-up state
  double ax2[2], ae2[2];        // level M-2 accumulators (X: [1,1] rows; Y/Z: [1,2,1] rows)
  double ax3 = 0.0, ae3 = 0.0;  // level c accumulators
#pragma unroll
  for (int k = 0; k < 2; ++k) ax2[k] = ae2[k] = 0.0;
  constexpr long long OP1 = 1ll << (2 * (M - 1)), OP2 = 1ll << (2 * (M - 2)), OP3 = 1ll << (2 * C);
  const double sc1 = p2d(-(M - 1)), sc2 = p2d(-(M - 2)), sc3 = p2d(-C);
  const int own1_end = I0 + RB, own2_end = (I0 + RB) >> 1, own3_end = (I0 + RB) >> 2;
  const bool emit1 = (M - 1) < oband, emit2 = (M - 2) < oband, emit3 = C < oband;

  // level M-2 row i2 complete (2 columns per lane) -> level c
  auto on_m2 = [&](int i2, const double (&Gm)[2]) {
    const double nb = __shfl_sync(FULL, Gm[0], Lg + 1, LPR);
    if (FLD == 0) {
      const double h = Gm[0] + 2.0 * Gm[1] + nb;
      if ((i2 & 1) == 0) {
        ax3 = h;
        ae3 = Gm[0];
      } else {
        const int i3 = i2 >> 1;
        wsS[(long long)FLD * HC * HC + (long long)i3 * HC + Lg] = 0.25 * (ax3 + h);
        if (emit3) out[OP3 * (1 + FLD) + (long long)i3 * HC + Lg] = (float)(0.25 * (ae3 + Gm[0]) * sc3);
      }
    } else {
      const double h = (FLD == 1) ? Gm[0] + Gm[1] : Gm[0] + 2.0 * Gm[1] + nb;
      if ((i2 & 1) == 0) {
        if (i2 > (I0 >> 1)) {
          const int i3 = (i2 >> 1) - 1;
          wsS[(long long)FLD * HC * HC + (long long)i3 * HC + Lg] = 0.25 * (ax3 + h);
        }
        ax3 = h;
        const int i3 = i2 >> 1;
        if (emit3 && i3 < own3_end) {
          const double d = (FLD == 1) ? Gm[0] + Gm[1] : Gm[0];
          out[OP3 * (1 + FLD) + (long long)i3 * HC + Lg] = (float)(0.25 * d * sc3);
        }
      } else {
        ax3 += 2.0 * h;
      }
    }
  };
  // level M-1 row i complete (CPL columns per lane) -> level M-2
  auto on_m1 = [&](int i, const double (&Fr)[CPL]) {
    const double nb = __shfl_sync(FULL, Fr[0], Lg + 1, LPR);
    double h[2];
    h[0] = (FLD == 1) ? Fr[0] + Fr[1] : Fr[0] + 2.0 * Fr[1] + Fr[2];
    h[1] = (FLD == 1) ? Fr[2] + Fr[3] : Fr[2] + 2.0 * Fr[3] + nb;
    if (FLD == 0) {
      if ((i & 1) == 0) {
        ax2[0] = h[0]; ax2[1] = h[1];
        ae2[0] = Fr[0]; ae2[1] = Fr[2];
      } else {
        const int i2 = i >> 1;
        double Gm[2] = {0.25 * (ax2[0] + h[0]), 0.25 * (ax2[1] + h[1])};
        if (emit2) {
          float2 v = make_float2((float)(0.25 * (ae2[0] + Fr[0]) * sc2), (float)(0.25 * (ae2[1] + Fr[2]) * sc2));
          *reinterpret_cast<float2*>(out + OP2 * (1 + FLD) + (long long)i2 * H2 + 2 * Lg) = v;
        }
        on_m2(i2, Gm);
      }
    } else {
      if ((i & 1) == 0) {
        if (i > I0) {
          double Gm[2] = {0.25 * (ax2[0] + h[0]), 0.25 * (ax2[1] + h[1])};
          on_m2((i >> 1) - 1, Gm);
        }
        ax2[0] = h[0]; ax2[1] = h[1];
        const int i2 = i >> 1;
        if (emit2 && i2 < own2_end) {
          const double d0 = (FLD == 1) ? Fr[0] + Fr[1] : Fr[0];
          const double d1 = (FLD == 1) ? Fr[2] + Fr[3] : Fr[2];
          *reinterpret_cast<float2*>(out + OP2 * (1 + FLD) + (long long)i2 * H2 + 2 * Lg) =
              make_float2((float)(0.25 * d0 * sc2), (float)(0.25 * d1 * sc2));
        }
      } else {
        ax2[0] += 2.0 * h[0];
        ax2[1] += 2.0 * h[1];
      }
    }
  };

  // ---------------------------------------------------------------- the stream: one parent row p per step
  const int nsteps = (FLD == 0) ? RB + 1 : RB + 4 + o;
  double c1[CPL], c2[CPL], vc[CPL];   // carries of the output rows in flight (X: c1 = X', c2 = H')
#pragma unroll
  for (int q = 0; q < CPL; ++q) c1[q] = c2[q] = vc[q] = 0.0;
  double Dp[3][W1D], Dq[3][W1D];
  if (FLD != 0) window1(pbase, Dq);

#pragma unroll 1
  for (int k = 0; k < nsteps; ++k) {
    const int p = pbase + k;
    if ((p >> 1) != cur_g) group1(p >> 1);
    double F1[W1F];
#pragma unroll
    for (int u = 0; u < W1F; ++u) F1[u] = (p & 1) ? F1g[W1F + u] : F1g[u];   // row 2 g2 + (p & 1)
    if (FLD == 0) {
      window1(p, Dp);
    } else {
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int u = 0; u < W1D; ++u) Dp[t][u] = Dq[t][u];
      window1(p + 1, Dq);
    }
    // the parent's two level-M child rows, horizontally filtered
    double hE[CPL], hO[CPL], gE[CPL], gO[CPL];
    {
      double x[NCE];
      children<FLD, 0, NCE>(F1, Dp, Dp, x);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int v = 0; v < NT; ++v) a = fma(TA[v], x[2 * q + v], a);
        if (FLD != 1) {
#pragma unroll
          for (int v = 0; v < 3; ++v) b = fma(TB[v], x[2 * q + v], b);
        }
        hE[q] = a;
        gE[q] = b;
      }
      children<FLD, 1, NCE>(F1, Dp, Dq, x);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int v = 0; v < NT; ++v) a = fma(TA[v], x[2 * q + v], a);
        if (FLD != 1) {
#pragma unroll
          for (int v = 0; v < 3; ++v) b = fma(TB[v], x[2 * q + v], b);
        }
        hO[q] = a;
        gO[q] = b;
      }
    }
    // vertical: the output row completed by this step, and the carries
    double done[CPL];
    if (FLD == 0) {
      const int ie = p + qh - 1 + o;   // X' / H' row completed
      double hv[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        done[q] = 0.25 * fma(ae, hE[q], fma(ao, hO[q], c1[q]));
        hv[q] = 0.25 * fma(ae, gE[q], fma(ao, gO[q], c2[q])) * sc1;
        c1[q] = fma(be, hE[q], bo * hO[q]);
        c2[q] = fma(be, gE[q], bo * gO[q]);
      }
      if (ie >= I0) {
        if (emit1)
          *reinterpret_cast<float4*>(out + OP1 * 1 + (long long)ie * H1 + 4 * Lg) =
              make_float4((float)hv[0], (float)hv[1], (float)hv[2], (float)hv[3]);
        on_m1(ie, done);
      }
    } else {
      const int ie = p + qh - 1;   // Y' / Z' row completed
      const int iv = p + qh;       // V^' / D^' row completed
      double hv[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const double se = (FLD == 1) ? hE[q] : gE[q], so = (FLD == 1) ? hO[q] : gO[q];
        done[q] = 0.25 * fma(ae, hE[q], fma(ao, hO[q], c1[q]));
        c1[q] = fma(be, hE[q], fma(bo, hO[q], c2[q]));
        c2[q] = fma(ge, hE[q], go * hO[q]);
        hv[q] = 0.25 * fma(ve, se, fma(vo, so, vc[q])) * sc1;
        vc[q] = vg * so;
      }
      if (emit1 && iv >= I0 && iv < own1_end)
        *reinterpret_cast<float4*>(out + OP1 * (1 + FLD) + (long long)iv * H1 + 4 * Lg) =
            make_float4((float)hv[0], (float)hv[1], (float)hv[2], (float)hv[3]);
      if (ie >= I0) on_m1(ie, done);
    }
  }
}

// One CTA: stage the band's rows (floats by cp.async into the upper half of the fp64 area, then
// widened in place to fp64 in averaging units), then one warp per field.
template <int M>
__device__ __forceinline__ void stream_cta(const ShiftArgs& args, const FaceParam& P, int g, unsigned char* smem) {
  using G = SG<M>;
  if ((int)blockIdx.x >= G::NBANDS) return;
  const int J0 = blockIdx.x * G::HB;
  constexpr int C = M - 3;
  // rows the CTA reads (stream_task): parents p = pbase .. pbase + RB + 4 + o of every row group and
  // p + 1; level M-2 rows p >> 1 and + 1; level c rows (p >> 1) >> 1 and + 1
  const int e1 = (-P.Qy - 1) >> 1;                   // pbase(I0) = I0 + e1
  const int first1 = J0 + e1, last1 = J0 + G::HB + e1 + 5;
  const RowSet R1 = make_rows(first1, last1, G::H1, G::NR1);
  const RowSet R2 = make_rows(first1 >> 1, ((last1 - 1) >> 1) + 1, G::H2, G::NR2);
  const RowSet R3 = make_rows(first1 >> 2, ((last1 - 1) >> 2) + 1, G::HC, G::NR3);
  const RowSet RW = make_rows(first1 >> 2, (last1 - 1) >> 2, G::HC, G::NRW);
  const int cq = -P.Qx - 1;
  const int s1 = (cq >> 1) & (G::H1 - 1), s2 = s1 >> 1, s3 = s2 >> 1;

  const int b_ = g / args.faces, f_ = g % args.faces;
  const float* __restrict__ in = args.in + (long long)b_ * args.in_batch_stride + (long long)f_ * args.in_face_stride;
  float* S = reinterpret_cast<float*>(smem);
  double* SW = reinterpret_cast<double*>(smem) + G::OFFW;
  constexpr long long L1 = 1ll << (2 * (M - 1)), L2 = 1ll << (2 * (M - 2)), L3 = 1ll << (2 * C);
  stage_rows<4, G::LPR, 1, G::ROW1, G::PLANE1>(in + L1, L1, R1, s1, S);
  stage_rows<2, G::LPR, 1, G::ROW2, G::PLANE2>(in + L2, L2, R2, s2, S + G::OFF2);
  stage_rows<1, G::LPR, 2, G::ROW3, G::PLANE3>(in + L3, L3, R3, s3, S + G::OFF3);
  const double* wsU = reinterpret_cast<const double*>(reinterpret_cast<const char*>(args.ws) +
                                                      (long long)g * args.ws_face_stride) + 3ll * G::HC * G::HC;
  stage_rows<1, G::LPR, 1, G::ROWW, G::PLANEW>(wsU, (long long)G::HC * G::HC, RW, s3, SW);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  switch (threadIdx.x >> 5) {
    case 0: stream_task<M, 0>(args, P, g, J0, S, SW, R1, R2, R3, RW); break;
    case 1: stream_task<M, 1>(args, P, g, J0, S, SW, R1, R2, R3, RW); break;
    default: stream_task<M, 2>(args, P, g, J0, S, SW, R1, R2, R3, RW); break;
  }
}

// grid: x = band (CTA of HB output rows at level m-1), y = face; warp = field.
__global__ void __launch_bounds__(kStreamThreads, 4) shift2d_stream_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char ssm[];
  const int g = blockIdx.y;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  if (blockIdx.x == 0 && threadIdx.x == 0 && stream_level(P.m)) {   // scaling coefficient: unchanged (R8)
    const int b_ = g / args.faces, f_ = g % args.faces;
    args.out[(long long)g * args.out_face_stride] =
        __ldg(args.in + (long long)b_ * args.in_batch_stride + (long long)f_ * args.in_face_stride);
  }
  switch (P.m) {
    case 6: stream_cta<6>(args, P, g, ssm); break;
    case 7: stream_cta<7>(args, P, g, ssm); break;
    case 8: stream_cta<8>(args, P, g, ssm); break;
    default: break;
  }
}

}  // namespace

// One CTA per (face, band of SG<m>::HB output rows): 8 bands for m = 8, 2 for m = 7, 1 for m = 6.
hs_status launch_shift2d_stream(ShiftArgs& a, cudaStream_t st) {
  HS_SMEM_ATTR(shift2d_stream_kernel, kStreamSmem);
  shift2d_stream_kernel<<<dim3(kStreamMaxBands, a.num_faces), kStreamThreads, kStreamSmem, st>>>(a);
  HS_CHECK_LAUNCH("shift2d_stream_kernel");
  return HS_OK;
}

}  // namespace hs
