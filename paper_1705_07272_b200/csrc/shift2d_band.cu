// 2D Haar-domain shift for working levels m = 6 .. 9 (every fractional shift at N = 64 .. 512; the
// c3, c5 and c5x configurations) -- SURVEY.md §8(a) rows a2-a4, DESIGN.md §4.1 "Band kernel".
//
// The paper's fields are finite differences of one function ("the horizontal, vertical, and
// diagonal coefficients are simply first order finite difference approximations"): X = A[i][j] -
// A[i][j+1], Y = A[i][j] - A[i+1][j], Z = X[i][j] - X[i+1][j] of the level-l approximation A.  The
// three field recursions of shift2d.cu (top-down eq:pde1-2 P:416-425 made exact, shift P:459 /
// P:508, bottom-up [1,1] (x) [1,2,1] / 4, eq:conv P:466-497) are therefore the recursions of
// A itself written on its differences, and this kernel carries A instead (one fp64 field where the
// difference form carries three; ~4x fewer fp64 operations per coefficient):
//   top-down   A_{l+1}[2i+a][2j+b] = A_l[i][j] + s_ab,  s_00 = H+V+D, s_01 = -H+V-D, s_10 = H-V-D,
//              s_11 = -H-V+D (details in averaging units, 2^l x unit); A_0 = 0 -- the scaling
//              coefficient drops out of every difference, as X_0 = Y_0 = Z_0 = 0 in the paper's form;
//   shift      A'[r][c] = sum_{a,b in {0,1}} w^y_a w^x_b A[r - Qy - a][c - Qx - b] at level m
//              (w_1 = phi, w_0 = 1 - phi: the same box weights the fields take);
//   bottom-up  the Haar analysis of A': H' = (a00 - a01 + a10 - a11) / 4 etc. -- exactly the
//              paper's  H'_l = (X'[2i][2j] + X'[2i+1][2j]) / 4  and  X'_l = [1,1] (x) [1,2,1] / 4
//              X'_{l+1} written on A' (DESIGN.md §4.1 derives the identity); the oracle keeps the
//              difference form, so the parity tests check the identity too.
// Periodic in rows and columns at every level, as the fields are.
//
//   shift2d_band_kernel   one CTA (8 warps) per (face, band of kBH = 16 output rows at level m).
//                         Loads (one round trip): the detail rows its shifted window needs at levels
//                         0 .. m-2 by cp.async into shared memory (fp32), level m-1's straight into
//                         registers.  Top-down 0 -> m in fp64 shared memory (levels < m-4: two rows;
//                         then exactly (16 >> (m-l)) + 1 rows of 2^l columns; 18 rows of 2^m at m).
//                         Shift + analysis m -> m-4 with one thread per output COLUMN streaming the
//                         17 source rows (conflict-free shared loads, lanes = consecutive columns):
//                         rows pair in time, columns pair across lanes (shuffles with lanes c^1, c^2,
//                         c^4, c^8), so the whole analysis stays in registers.  Details of levels
//                         m-1 .. m-4 go to the output (levels below the band only), the band's one
//                         row of A'_{m-4} to the workspace.  54 KB shared memory at m = 8: 4 CTAs/SM.
//   band_finish_kernel    one CTA per face: the analysis of A'_{m-4} (2^(m-4) squared) down to
//                         level 0, and the scaling coefficient (unchanged by a shift, R8).
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

constexpr int kBH = 16;          // output rows at level m per CTA
constexpr int kBandThreads = 256;
constexpr int kKF = 4;           // levels per band: the band kernel starts from A_L, L = m - kKF

__device__ __forceinline__ double p2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}

// Band geometry at working level M.  Level l in [L, M) (L = M - 4): the band reads the detail rows
// [Slo >> (M - l), Shi >> (M - l)] -- exactly NR(l) = (kBH >> (M - l)) + 1 rows of 2^l columns (the
// window spans kBH + 1 rows at level M); levels l < L: 1 or 2 rows, always staged and expanded as 2.
// Shared memory (doubles): level M rows (18 x W), levels M-1 / M-3 (5 W), the coarse levels' ping-pong
// (2 x 4 x W / 16), then the staged fp32 detail rows of levels 0 .. M-2 (level M-1's details go
// straight to registers: no shared-memory copy for the largest level).
template <int M>
struct BG {
  static constexpr int W = 1 << M, L = M - kKF, WL = W >> kKF, NBANDS = W / kBH;
  static constexpr int NR(int l) { return l < L ? 2 : (kBH >> (M - l)) + 1; }
  static constexpr int SOFF(int l) {   // float offset of level l's staged rows (3 planes each)
    int o = 0;
    for (int k = 0; k < l; ++k) o += ((3 * NR(k) * (1 << k) + 3) & ~3);
    return o;
  }
  static constexpr int STAGE = SOFF(M - 1);
  static constexpr int OFF_B = 18 * W, OFF_C = OFF_B + 5 * W, OFF_S = OFF_C + 8 * WL;   // doubles
  static constexpr size_t SMEM = (size_t)OFF_S * 8 + (size_t)STAGE * 4;
  static constexpr int KP = (NR(M - 1) * (W / 2) + kBandThreads - 1) / kBandThreads;   // level M-1 parents per thread
};
constexpr size_t band_smem_bytes(int m) {
  return m == 6 ? BG<6>::SMEM : m == 7 ? BG<7>::SMEM : m == 8 ? BG<8>::SMEM : BG<9>::SMEM;
}

// forward Haar step of a 2 x 2 block (averaging units): returns the average, writes the details
__device__ __forceinline__ double analyse(double s00, double s01, double s10, double s11, double& H, double& V,
                                          double& D) {
  const double p = s00 + s01, q = s10 + s11, u = s00 - s01, v = s10 - s11;
  H = 0.25 * (u + v);
  V = 0.25 * (p - q);
  D = 0.25 * (u - v);
  return 0.25 * (p + q);
}

// Top-down step level l -> l + 1 over the NRL parent rows from `lo` (stored from row `pbase` in P):
// children rows from 2 lo in C; details from the staged rows S (3 planes of NRL x 2^l floats).
template <int l, int NRL>
__device__ __forceinline__ void topdown_step(const double* __restrict__ P, int pbase, int lo,
                                             const float* __restrict__ S, double* __restrict__ C) {
  constexpr int gl = 1 << l;
  constexpr float asc = float(1u << l);   // unit -> averaging, exact in fp32 (|d| < 2^100)
  const double* Pr = P + (lo - pbase) * gl;
#pragma unroll 2
  for (int idx = threadIdx.x; idx < NRL * gl; idx += kBandThreads) {
    const int rr = idx >> l, j = idx & (gl - 1);
    const double a = Pr[idx];
    const float* sd = S + idx;
    const double H = (double)(sd[0] * asc), V = (double)(sd[NRL * gl] * asc), D = (double)(sd[2 * NRL * gl] * asc);
    const double p = a + V, q = a - V, s = H + D, t = H - D;
    double* c0 = C + (2 * rr) * (2 * gl) + 2 * j;
    *reinterpret_cast<double2*>(c0) = make_double2(p + s, p - s);
    *reinterpret_cast<double2*>(c0 + 2 * gl) = make_double2(q + t, q - t);
  }
}

// One analysis step across lanes: the 2 x 2 block of rows (in time) x columns (lanes c, c ^ X) from
// this lane's column sums e = s_top + s_bottom and differences d = s_top - s_bottom.  The block's
// left lane gets the average and H, the right lane V and D.
template <int X>
__device__ __forceinline__ void lane_analyse(double e, double d, bool right, double& sum, double& dif) {
  // Unscaled (x 4 per level; the factors are folded into the emission scales): the block's left
  // lane gets sum = e_l + e_r (4 avg) and dif = e_l - e_r (4 H); the right lane sum = d_l + d_r
  // (4 V) and dif = d_r - d_l (-4 D: the sign is folded into the right lanes' scale).
  const double own = right ? d : e;
  const double r = __shfl_xor_sync(0xffffffffu, right ? e : d, X);
  sum = own + r;
  dif = own - r;
}

// Emission of one analysis block's details: the left lane writes H (plane 1), the right lane V
// (plane 2) and D (plane 3) -- one store per lane plus one predicated store, no divergent branch.
__device__ __forceinline__ void emit(float* __restrict__ base, long long per, bool right, double sum, double dif,
                                     double sc, double scd) {
  const float v1 = (float)((right ? sum : dif) * sc);
  float* p1 = right ? base + 2 * per : base + per;
  *p1 = v1;
  if (right) base[3 * per] = (float)(dif * scd);
}

// The last step M-1 -> M with the details already in registers (dr[k][t] for parent tid + k T).
template <int l, int NRL, int KP>
__device__ __forceinline__ void topdown_last(const double* __restrict__ P, int pbase, int lo, const float (&dr)[KP][3],
                                             double* __restrict__ C) {
  constexpr int gl = 1 << l;
  constexpr float asc = float(1u << l);
  const double* Pr = P + (lo - pbase) * gl;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int idx = threadIdx.x + k * kBandThreads;
    if (idx < NRL * gl) {
      const int rr = idx >> l, j = idx & (gl - 1);
      const double a = Pr[idx];
      const double H = (double)(dr[k][0] * asc), V = (double)(dr[k][1] * asc), D = (double)(dr[k][2] * asc);
      const double p = a + V, q = a - V, s = H + D, t = H - D;
      double* c0 = C + (2 * rr) * (2 * gl) + 2 * j;
      *reinterpret_cast<double2*>(c0) = make_double2(p + s, p - s);
      *reinterpret_cast<double2*>(c0 + 2 * gl) = make_double2(q + t, q - t);
    }
  }
}

// Stage level l's detail rows (NR(l) rows from Slo >> (M - l), 3 planes) -- compile-time l, so
// every index division is by a constant.
template <int M, int l>
__device__ __forceinline__ void stage_level(const float* __restrict__ in, int Slo, bool al16, float* __restrict__ stage) {
  using G = BG<M>;
  constexpr int gl = 1 << l, nr = G::NR(l);
  constexpr long long per = 1ll << (2 * l);
  const int llo = Slo >> (M - l);
  float* S = stage + G::SOFF(l);
  bool done = false;
  if constexpr (l >= 2) {
    if (al16) {
      constexpr int q = gl / 4;                     // 16-byte chunks per row
      for (int idx = threadIdx.x; idx < 3 * nr * q; idx += kBandThreads) {
        const int row = idx / q, c4 = idx - row * q;   // row = t * nr + rr
        const int t = row / nr, rr = row - t * nr;
        cp_async16(S + row * gl + 4 * c4, in + per * (1 + t) + (long long)((llo + rr) & (gl - 1)) * gl + 4 * c4);
      }
      done = true;
    }
  }
  if (!done) {
    for (int idx = threadIdx.x; idx < 3 * nr * gl; idx += kBandThreads) {
      const int row = idx >> l, c = idx & (gl - 1);
      const int t = row / nr, rr = row - t * nr;
      cp_async4(S + idx, in + per * (1 + t) + (long long)((llo + rr) & (gl - 1)) * gl + c);
    }
  }
  if constexpr (l + 1 < M - 1) stage_level<M, l + 1>(in, Slo, al16, stage);
}

// Levels l .. L-1 of the top-down on one warp (two parent rows per level, at most 2 x 2^(L-1)
// parents: warp-synchronous, no block barrier); returns the first stored row of level L.
template <int M, int l>
__device__ __forceinline__ int coarse_levels(const float* __restrict__ stage, int Slo, int base, double* cur,
                                             double* nxt) {
  using G = BG<M>;
  constexpr int L = G::L;
  if constexpr (l == L) {
    return base;
  } else {
    constexpr int gl = 1 << l;
    constexpr float asc = float(1u << l);
    const int lane = threadIdx.x & 31;
    const int lo = Slo >> (M - l);
    const float* S = stage + G::SOFF(l);
    for (int idx = lane; idx < 2 * gl; idx += 32) {
      const int rr = idx >> l, j = idx & (gl - 1);
      const double a = cur[(lo + rr - base) * gl + j];
      const double H = (double)(S[idx] * asc), V = (double)(S[2 * gl + idx] * asc), D = (double)(S[4 * gl + idx] * asc);
      const double p = a + V, q = a - V, sm = H + D, t = H - D;
      double* c0 = nxt + (2 * rr) * (2 * gl) + 2 * j;
      c0[0] = p + sm;
      c0[1] = p - sm;
      c0[2 * gl] = q + t;
      c0[2 * gl + 1] = q - t;
    }
    __syncwarp();
    return coarse_levels<M, l + 1>(stage, Slo, 2 * lo, nxt, cur);
  }
}

template <int M>
__device__ __forceinline__ void band_cta(const ShiftArgs& args, const FaceParam& P, int g, double* smem) {
  using G = BG<M>;
  constexpr int W = G::W, L = G::L, WL = G::WL;
  if ((int)blockIdx.x >= G::NBANDS) return;
  const int tid = threadIdx.x;
  const int R0 = blockIdx.x * kBH;                  // output rows R0 .. R0 + 15 at level M
  const int Qy = P.Qy, Qx = P.Qx;
  const int Slo = R0 - Qy - 1;                      // source rows Slo .. Slo + 16 at level M (unwrapped)
  const int b_ = g / args.faces, f_ = g % args.faces;
  const float* __restrict__ in = args.in + (long long)b_ * args.in_batch_stride + (long long)f_ * args.in_face_stride;
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  double* const wsA = reinterpret_cast<double*>(reinterpret_cast<char*>(args.ws) + (long long)g * args.ws_face_stride);
  const int oband = args.band;
  double* const bufA = smem;                       // levels M, M-2
  double* const bufB = smem + G::OFF_B;            // levels M-1, M-3
  double* const sC = smem + G::OFF_C;              // levels 0 .. L (ping-pong, 4 rows x 2^l each)
  float* const stage = reinterpret_cast<float*>(smem + G::OFF_S);

  // ------------------------------------------------------------------ loads (one round trip)
  // level M-1 details -> registers (coalesced rows; consumed by the last top-down step)
  float dr[G::KP][3];
  {
    constexpr int l = M - 1, gl = 1 << l;
    const int llo = Slo >> 1;
    const long long per = 1ll << (2 * l);
#pragma unroll
    for (int k = 0; k < G::KP; ++k) {
      const int idx = tid + k * kBandThreads;
      if (idx < G::NR(l) * gl) {
        const int rr = idx >> l, j = idx & (gl - 1);
        const float* src = in + per + (long long)((llo + rr) & (gl - 1)) * gl + j;
        dr[k][0] = __ldg(src);
        dr[k][1] = __ldg(src + per);
        dr[k][2] = __ldg(src + 2 * per);
      }
    }
  }
  // levels 0 .. M-2 -> shared memory (cp.async)
  {
    const bool al16 = ((reinterpret_cast<unsigned long long>(in) & 15) == 0);
    stage_level<M, 0>(in, Slo, al16, stage);
    if (tid < 2) sC[tid] = 0.0;                      // A_0 = 0 (rows lo_0, lo_0 + 1 of level 0)
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }

  // ------------------------------------------------------------------ top-down 0 -> M
  // levels 0 .. L-1 on warp 0 (two parent rows from lo_l each, ping-pong in sC); A_0 = 0
  double* const cL = (L & 1) ? sC + 4 * WL : sC;      // where level L lands after L ping-pongs
  if (tid < 32) coarse_levels<M, 0>(stage, Slo, Slo >> M, sC, sC + 4 * WL);
  const int base = 2 * (Slo >> (M - L + 1));          // level L's first stored row (2 lo_{L-1})
  __syncthreads();
  double* cur = cL;
  // levels L .. M-1 (exact row counts)
  const int lo0 = Slo >> 4, lo1 = Slo >> 3, lo2 = Slo >> 2, lo3 = Slo >> 1;
  topdown_step<L, G::NR(L)>(cur, base, lo0, stage + G::SOFF(L), bufB);
  __syncthreads();
  topdown_step<L + 1, G::NR(L + 1)>(bufB, 2 * lo0, lo1, stage + G::SOFF(L + 1), bufA);
  __syncthreads();
  topdown_step<L + 2, G::NR(L + 2)>(bufA, 2 * lo1, lo2, stage + G::SOFF(L + 2), bufB);
  __syncthreads();
  topdown_last<L + 3, G::NR(L + 3), G::KP>(bufB, 2 * lo2, lo3, dr, bufA);
  __syncthreads();

  // ------------------------------------------------------------------ shift + analysis M -> L
  // One thread per output column c (lanes = consecutive columns), streaming the 17 source rows:
  // h = the horizontal taps of a source row, s = the vertical taps of two h rows = A'[R0 + r][c].
  // The analysis pairs rows in time (in the thread) and columns across lanes (lane_analyse), level
  // by level: lanes c ^ 1, c ^ 2, c ^ 4, c ^ 8 -- every value stays in registers.
  const double wy1 = (double)P.wy, wy0 = 1.0 - wy1, wx1 = (double)P.wx, wx0 = 1.0 - wx1;
  constexpr int CPT = W >= kBandThreads ? W / kBandThreads : 1;
  if (tid < W) {
    const double* rows = bufA + (Slo - 2 * lo3) * W;   // source row Slo (0 or 1 rows into the buffer)
    // emission scales: level M-k values are 4^k x (averaging units), output = unit = x 2^-(level)
    const double sc1 = p2d(-(M + 1)), sc2 = p2d(-(M + 2)), sc3 = p2d(-(M + 3)), sc4 = p2d(-(M + 4));
#pragma unroll 1
    for (int cc = 0; cc < CPT; ++cc) {
      const int c = tid + cc * kBandThreads;
      const bool r1 = (c & 1) != 0, r2 = (c & 2) != 0, r4 = (c & 4) != 0, r8 = (c & 8) != 0;
      const int ca = (c - Qx) & (W - 1), cb = (c - Qx - 1) & (W - 1);
      // output base of this lane's level M-1 block column (plane 0 offset; emit adds the planes)
      float* const o1 = out + (R0 >> 1) * (W >> 1) + (c >> 1);
      double hprev = fma(wx0, rows[ca], wx1 * rows[cb]);
      double s_top = 0.0;                        // level M row 2i of the pair in flight
      double a1_top = 0.0, a2_top = 0.0, a3_top = 0.0;   // levels M-1, M-2, M-3 pending rows
#pragma unroll
      for (int r = 0; r < kBH; ++r) {
        const double* rw = rows + (r + 1) * W;
        const double hcur = fma(wx0, rw[ca], wx1 * rw[cb]);
        const double sv = fma(wy0, hcur, wy1 * hprev);
        hprev = hcur;
        if ((r & 1) == 0) {
          s_top = sv;
          continue;
        }
        // level M-1 block (row pair i = r / 2, column pair c >> 1)
        const int i1 = r >> 1;
        double x1, y1;
        lane_analyse<1>(s_top + sv, s_top - sv, r1, x1, y1);
        if ((M - 1) < oband) emit(o1 + i1 * (W >> 1), 1ll << (2 * (M - 1)), r1, x1, y1, sc1, -sc1);
        if ((i1 & 1) == 0) {
          a1_top = x1;
          continue;
        }
        // level M-2 (lanes c ^ 2; valid in lanes with c % 2 == 0)
        const int i2 = i1 >> 1;
        double x2, y2;
        lane_analyse<2>(a1_top + x1, a1_top - x1, r2, x2, y2);
        if ((M - 2) < oband && !r1) emit(out + ((R0 >> 2) + i2) * (W >> 2) + (c >> 2), 1ll << (2 * (M - 2)), r2, x2, y2, sc2, -sc2);
        if ((i2 & 1) == 0) {
          a2_top = x2;
          continue;
        }
        // level M-3 (lanes c ^ 4; valid in lanes with c % 4 == 0)
        const int i3 = i2 >> 1;
        double x3, y3;
        lane_analyse<4>(a2_top + x2, a2_top - x2, r4, x3, y3);
        if ((M - 3) < oband && (c & 3) == 0)
          emit(out + ((R0 >> 3) + i3) * (W >> 3) + (c >> 3), 1ll << (2 * (M - 3)), r4, x3, y3, sc3, -sc3);
        if ((i3 & 1) == 0) {
          a3_top = x3;
          continue;
        }
        // level M-4 = L (lanes c ^ 8; valid in lanes with c % 8 == 0): one row per band
        double x4, y4;
        lane_analyse<8>(a3_top + x3, a3_top - x3, r8, x4, y4);
        if ((c & 7) == 0) {
          if (!r8) wsA[(long long)(R0 >> 4) * WL + (c >> 4)] = x4 * p2d(-8);   // A'_L (x 4^-4)
          if (L < oband) emit(out + (R0 >> 4) * WL + (c >> 4), 1ll << (2 * L), r8, x4, y4, sc4, -sc4);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kBandThreads, 4) shift2d_band_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char bsm[];
  const int g = blockIdx.y;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  double* smem = reinterpret_cast<double*>(bsm);
  switch (P.m) {
    case 6: band_cta<6>(args, P, g, smem); break;
    case 7: band_cta<7>(args, P, g, smem); break;
    case 8: band_cta<8>(args, P, g, smem); break;
    case 9: band_cta<9>(args, P, g, smem); break;
    default: break;
  }
  // programmatic dependent launch: band_finish_kernel may be scheduled once every band CTA got
  // here (it waits for this grid's completion and memory before reading the workspace)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Levels m-5 .. 0 of one face from A'_{m-4} (the bands' rows in the workspace), and the scaling
// coefficient.  At most 32 x 32 values: ping-pong in static shared memory.
__global__ void __launch_bounds__(kBandThreads) band_finish_kernel(const __grid_constant__ ShiftArgs args) {
  __shared__ double sA[32 * 32 + 16 * 16];
  const int g = blockIdx.x;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  if (!band_level(P.m)) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the band kernel's rows of A'_L are complete
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  if (threadIdx.x == 0) {   // scaling coefficient: unchanged (R8)
    const int b_ = g / args.faces, f_ = g % args.faces;
    out[0] = __ldg(args.in + (long long)b_ * args.in_batch_stride + (long long)f_ * args.in_face_stride);
  }
  const int L = P.m - kKF;
  const double* wsA = reinterpret_cast<const double*>(reinterpret_cast<const char*>(args.ws) + (long long)g * args.ws_face_stride);
  const int gL = 1 << L;
  for (int idx = threadIdx.x; idx < gL * gL; idx += blockDim.x) sA[idx] = __ldcg(wsA + idx);
  __syncthreads();
  double* src = sA;
  double* dst = sA + 32 * 32;
  for (int lv = L - 1; lv >= 0; --lv) {
    const int wl = 1 << lv;
    const long long per = 1ll << (2 * lv);
    const bool emit = lv < args.band;
    const double sc = p2d(-lv);
    for (int idx = threadIdx.x; idx < wl * wl; idx += blockDim.x) {
      const int i = idx >> lv, j = idx & (wl - 1);
      const double* s0 = src + (2 * i) * (2 * wl) + 2 * j;
      double H, V, D;
      dst[idx] = analyse(s0[0], s0[1], s0[2 * wl], s0[2 * wl + 1], H, V, D);
      if (emit) {
        out[per + idx] = (float)(H * sc);
        out[2 * per + idx] = (float)(V * sc);
        out[3 * per + idx] = (float)(D * sc);
      }
    }
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
}

}  // namespace

// grid (bands of the largest working level present, faces); faces at other levels exit at once.
hs_status launch_shift2d_band(ShiftArgs& a, int max_m, cudaStream_t st) {
  if (max_m < kBandMinLevel) return HS_OK;
  if (max_m > kBandMaxLevel) max_m = kBandMaxLevel;
  const size_t smem = band_smem_bytes(max_m);
  HS_SMEM_ATTR(shift2d_band_kernel, band_smem_bytes(kBandMaxLevel));
  shift2d_band_kernel<<<dim3((1u << max_m) / kBH, a.num_faces), kBandThreads, smem, st>>>(a);
  HS_CHECK_LAUNCH("shift2d_band_kernel");
  {   // programmatic dependent launch: its launch overlaps the band kernel's last wave
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.num_faces);
    cfg.blockDim = dim3(kBandThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HS_CHECK_CUDA(cudaLaunchKernelEx(&cfg, band_finish_kernel, a), "cudaLaunchKernelEx(band_finish_kernel)");
  }
  HS_CHECK_LAUNCH("band_finish_kernel");
  return HS_OK;
}

}  // namespace hs
