// 2D Haar-domain shift: exact difference-domain form of the paper's
// "coefficients are finite differences" relations, tiled for sm_100a.  DESIGN.md §4.1.
//
// Notation: averaging details H^,V^,D^ = 2^l * unit-square; fields of the approximation A_l at
// level l (periodic):
//   X_l[i][j] = A[i][j] - A[i][j+1]                 (horizontal difference ~ df/dphi,  P:415)
//   Y_l[i][j] = A[i][j] - A[i+1][j]                 (vertical difference   ~ df/dtheta)
//   Z_l[i][j] = A[i][j] - A[i][j+1] - A[i+1][j] + A[i+1][j+1]   (mixed, d2f/dphi dtheta)
// Children of cell (i,j): A_{l+1}[2i+a][2j+b] = A_l + delta_ab,
//   delta00 = H+V+D, delta01 = -H+V-D, delta10 = H-V-D, delta11 = -H-V+D.
//
//  (1) top-down, from the DETAIL coefficients only (no scaling coefficient, no pixel values):
//        X_{l+1}[2i+a][2j]   = d_a0(i,j) - d_a1(i,j)
//        X_{l+1}[2i+a][2j+1] = X_l[i][j] + d_a1(i,j) - d_a0(i,j+1)          (and Y, Z alike)
//      -- P:331/P:408/P:463 made exact: the level-(l+1) finite differences need the level-l
//         differences plus the neighbours' details (R13).
//  (2) shift at the working level m: every field translates (eq:pde1-2 P:416-425 with the
//      identity Jacobian of a pure shift):
//        F'_m[r][c] = sum_{a,b in {0,1}} w^y_a w^x_b F_m[r - Qy - a][c - Qx - b],  w0 = 1-phi, w1 = phi.
//  (3) bottom-up with the paper's 2-tap box h_s = [1,1] and 3-tap tent h_t = [1,2,1], decimated
//      by 2 (eq:conv/eq:tker/eq:sker P:466-478, recursive form P:486-497):
//        X'_l = 1/4 [1,1]_y (x) [1,2,1]_x X'_{l+1} |v2,  H^'_l = (X'_{l+1}[2i][2j] + X'_{l+1}[2i+1][2j]) / 4
//        Y'_l = 1/4 [1,2,1]_y (x) [1,1]_x Y'_{l+1} |v2,  V^'_l = (Y'_{l+1}[2i][2j] + Y'_{l+1}[2i][2j+1]) / 4
//        Z'_l = 1/4 [1,2,1] (x) [1,2,1] Z'_{l+1} |v2,     D^'_l = Z'_{l+1}[2i][2j] / 4
//      Steps (2) and the first step of (3) are fused into one separable stencil on F_m.
//
// Three launches per call:
//   coarse_fields_kernel  one CTA per face: (1) top-down over the full grid to the tile-root level
//                         c = max(0, m - KF) -> the unshifted level-c fields (workspace);
//   shift2d_tile_kernel   a CTA owns a TC x TC tile at level c and every output coefficient below
//                         it at levels c..m-1: it fetches its window of the level-c fields and the
//                         detail windows of levels c..m-1 with cp.async (one latency round trip),
//                         runs (1)-(3) over its window (all periodic index arithmetic on unwrapped
//                         coordinates), writes its outputs and its shifted level-c fields;
//   coarse_finish_kernel  one CTA per face: the coarse bottom-up c -> 0 from the shifted fields.
// Levels >= m (dyadic shifts) are exact permutations (permute_kernel).
//
// Field precision: fp64 at every size (DESIGN.md §4.1 error model: fine-level fp32 rounding is
// amplified ~2^(n-l) on the coarse outputs; at N = 256 the relight band of the c5 light reached
// 1.3e-5 per frame in fp32, 3e-8 in fp64; white noise at N = 64 with a one-level band 2e-5).
#include <cuda_runtime.h>

#include "common.cuh"

#ifdef HS_PHASE_TIMING  // debug builds only: per-CTA clock64 at phase boundaries
__device__ long long g_phase[1 << 18];
#define HS_PHASE(k)                                                                                   \
  if (threadIdx.x == 0 && ((long long)blockIdx.y * gridDim.x + blockIdx.x) < (1 << 14))             \
    hs::g_phase_ptr()[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (k)] = clock64();
namespace hs {
__device__ __forceinline__ long long* g_phase_ptr() { return g_phase; }
}
extern "C" HS_API int hs_debug_phase_dump(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_phase, (size_t)n * sizeof(long long));
}
#else
#define HS_PHASE(k)
#endif

namespace hs {
namespace {

constexpr int KF = kTileKF;
constexpr int TC = kTileTC;
constexpr int kThreads = 256;
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
template <typename FT>
__device__ __forceinline__ void cp_async_ft(FT* dst, const FT* src) {
  if constexpr (sizeof(FT) == 8) cp_async8(dst, src); else cp_async4(dst, src);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Exact 2^e for |e| < 127 (no libm call).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// floor(x / n) for 0 <= x < 2^16, 1 <= n < 2^10 from an approximate reciprocal: (x + 1/2)/n is at
// least 1/(2n) away from an integer and the float error is < 2^-21 * 2^16 / n, so the floor is exact.
__device__ __forceinline__ int div_small(int x, float inv_n) { return __float2int_rd(((float)x + 0.5f) * inv_n); }
__device__ __forceinline__ float inv_small(int n) { return __fdividef(1.0f, (float)n); }

// Coarse bottom-up of one face from the shifted level-c fields (periodic full grid) to level 0.
// src/dst may point to shared or global memory (generic addressing); global reads use ld.cg.
template <typename FT>
__device__ void coarse_finish(const FT* src0, FT* b0, FT* b1, int c, float* __restrict__ out, int band,
                              bool global) {
  const FT* src = src0;
  FT* dst = b0;
  const FT q = FT(0.25);
  for (int lev = c - 1; lev >= 0; --lev) {
    const int g = 1 << lev, G = 2 * g, GG = G * G, gg = g * g;
    const FT sc = FT(pow2f(-lev));
    for (int idx = threadIdx.x; idx < gg; idx += blockDim.x) {
      const int i = idx >> lev, j = idx & (g - 1);
      const int rr[3] = {2 * i, 2 * i + 1, (2 * i + 2) & (G - 1)};
      const int cc[3] = {2 * j, 2 * j + 1, (2 * j + 2) & (G - 1)};
      FT v[3][3][3];
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int u = 0; u < 3; ++u)
#pragma unroll
          for (int w = 0; w < 3; ++w) {
            const FT* p = src + f * GG + rr[u] * G + cc[w];
            v[f][u][w] = global ? __ldcg(p) : *p;
          }
      dst[idx] = q * (v[0][0][0] + FT(2) * v[0][0][1] + v[0][0][2] + v[0][1][0] + FT(2) * v[0][1][1] + v[0][1][2]);
      dst[gg + idx] =
          q * (v[1][0][0] + FT(2) * v[1][1][0] + v[1][2][0] + v[1][0][1] + FT(2) * v[1][1][1] + v[1][2][1]);
      dst[2 * gg + idx] = q * ((v[2][0][0] + FT(2) * v[2][0][1] + v[2][0][2]) +
                               FT(2) * (v[2][1][0] + FT(2) * v[2][1][1] + v[2][1][2]) +
                               (v[2][2][0] + FT(2) * v[2][2][1] + v[2][2][2]));
      if (lev < band) {
        out[(long long)gg * 1 + idx] = (float)(q * (v[0][0][0] + v[0][1][0]) * sc);
        out[(long long)gg * 2 + idx] = (float)(q * (v[1][0][0] + v[1][0][1]) * sc);
        out[(long long)gg * 3 + idx] = (float)(q * v[2][0][0] * sc);
      }
    }
    __syncthreads();
    src = dst;
    dst = (dst == b0) ? b1 : b0;
  }
}

// ------------------------------------------------------------------------------------------
// Compile-time tile geometry for K fine levels below a TC x TC tile at the tile-root level c.
// d = m - l counts levels above the working level m.  Window sides are maxima (the actual
// windows, whose starts are runtime, fit inside; extra cells are computed from valid periodic
// data and never written out).
template <int K, int TC>
struct TGeo {
  static constexpr int FW = (TC + 1) << K;                    // level-m field window
  static constexpr int P(int d) {                              // parent window at level m-d
    int s = FW;
    for (int i = 0; i < d; ++i) s = s / 2 + 1;
    return s;
  }
  static constexpr int P1 = P(1);                              // parents at level m-1
  static constexpr int CH = 2 * P1;                            // level-m children side
  static constexpr int HC = P1;                                // parity half row
  static constexpr int CB = 2 * P(2);                          // level m-1 field side
  static constexpr int SN(int e) { return ((TC + 1) << e) - 1; }  // shifted window at c+e
  static constexpr int SN1 = SN(K - 1);
  static constexpr int NSTRIP = (kThreads / SN1 < SN1) ? kThreads / SN1 : SN1;
  static constexpr int RSS = (SN1 + NSTRIP - 1) / NSTRIP;      // fused-stencil rows per strip
  static constexpr int CHR = CH + 2 * (NSTRIP * RSS - SN1);     // child plane rows incl. spare
  static constexpr int DETW(int d) { return P(d) + 1; }
  static constexpr int WS1 = (DETW(1) + 6 + 3) / 4 * 4;  // padded row of the level m-1 window (16B chunks)
  static constexpr int DET_MAX = [] {
    int o = 3 * DETW(1) * WS1;
    for (int d = 2; d <= HS_MAX_LOG2N; ++d) o += 3 * DETW(d) * DETW(d);
    return o;
  }();
  static constexpr int ANC_MAX = 2 * P(3) > 2 * P(4) ? 2 * P(3) : 2 * P(4);  // level <= m-2 side
};

template <typename FT, int K, int TC>
struct TSmem {
  using G = TGeo<K, TC>;
  static constexpr int DET = 0;                                                      // float
  static constexpr int B1 = (DET + G::DET_MAX * 4 + 15) / 16 * 16;                   // FT[3][CB^2]
  static constexpr int CHILD = B1 + 3 * G::CB * G::CB * (int)sizeof(FT);             // FT[2][CHR][HC], one field
  // the child plane also holds the two ancestor-field halves (3 ANC_MAX^2 each) before step (1')
  static constexpr int CHILD_ELEMS = (2 * G::CHR * G::HC > 6 * G::ANC_MAX * G::ANC_MAX) ? 2 * G::CHR * G::HC
                                                                                       : 6 * G::ANC_MAX * G::ANC_MAX;
  static constexpr int BYTES = CHILD + CHILD_ELEMS * (int)sizeof(FT);
  static_assert(3 * G::SN1 * G::SN1 <= 3 * G::CB * G::CB, "shifted m-1 window aliases B1");
};

// Detail windows of levels l = m - d for d in [D, DEND] (d <= m): [3][W][W] floats each with the
// compile-time side W = P(d) + 1, gathered element-wise (periodic) with cp.async.
template <class G, int D, int DEND>
__device__ __forceinline__ void load_windows(const float* __restrict__ in, float* sDet,
                                             const int (*sR)[2][HS_MAX_LOG2N + 1], const int* sDoff, int m) {
  if constexpr (D <= DEND) {
    if (D <= m) {
      constexpr int W = G::DETW(D), PER = W * W;
      const int l = m - D;
      const int ys = sR[0][0][l], xs = sR[1][0][l], mask = (1 << l) - 1;
      float* dst = sDet + sDoff[l];
      for (int e = threadIdx.x; e < 3 * PER; e += kThreads) {
        const int t = e / PER, rem = e - t * PER;
        const int a = rem / W, bb = rem - a * W;
        cp_async4(dst + e, in + (((1 + t) << (2 * l)) + (((ys + a) & mask) << l) + ((xs + bb) & mask)));
      }
      load_windows<G, D + 1, DEND>(in, sDet, sR, sDoff, m);
    }
  }
}

// Level m-1 window (d = 1) with 16-byte cp.async: every row covers the same (periodic) column
// range [xs, xs + W); it is stored with row stride WS1 at smem column (col - xs) + (xs & 3), so the
// aligned global chunks of both segments of a wrapping row land 16-byte aligned in smem.
template <class G>
__device__ __forceinline__ void load_window_vec(const float* __restrict__ in, float* sDet,
                                                const int (*sR)[2][HS_MAX_LOG2N + 1], const int* sDoff, int m) {
  constexpr int W = G::DETW(1), WS = G::WS1, NCH = WS / 4, ROWS = 3 * W;
  const int l = m - 1;
  const int gl = 1 << l, mask = gl - 1;
  const int ys = sR[0][0][l];
  const int xsm = sR[1][0][l] & mask;
  const int c0 = xsm & ~3;
  const bool wrap = xsm + W > gl;
  const int n1 = ((wrap ? gl : ((xsm + W + 3) & ~3)) - c0) >> 2;     // chunks of segment 1
  const int ntot = n1 + (wrap ? ((xsm + W - gl + 3) >> 2) : 0);
  float* dst = sDet + sDoff[l];
  for (int e = threadIdx.x; e < ROWS * NCH; e += kThreads) {
    const int row = e / NCH, k = e - row * NCH;
    if (k >= ntot) continue;
    const int t = row / W, a = row - t * W;
    const int col = (k < n1) ? c0 + 4 * k : 4 * (k - n1);
    const float* src = in + ((1 + t) << (2 * l)) + (((ys + a) & mask) << l) + col;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst + row * WS + 4 * k)),
                 "l"(src)
                 : "memory");
  }
}

template <typename FT, int K, int TC>
__device__ __forceinline__ void tile_body(const ShiftArgs& args, unsigned char* smem, const FaceParam& P, int g,
                                          int m, int c, int i0, int j0, int (*sR)[2][HS_MAX_LOG2N + 1],
                                          int* sDoff) {
  using G = TGeo<K, TC>;
  using S = TSmem<FT, K, TC>;
  constexpr int CB = G::CB, HC = G::HC, CHR = G::CHR, SN1 = G::SN1;
  constexpr int PLANE_C = CHR * HC;  // one parity plane of one field's children
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in =
      args.in + (long long)b * args.in_batch_stride + (long long)f * args.in_face_stride;
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  const int band = args.band;
  const int tid = threadIdx.x;
  float* sDet = reinterpret_cast<float*>(smem + S::DET);
  FT* sB1 = reinterpret_cast<FT*>(smem + S::B1);
  FT* sCh = reinterpret_cast<FT*>(smem + S::CHILD);

  HS_PHASE(0)
  // ---- window starts: level-m window [2^K i0 - Q - 1, + FW); level m-d starts at floor(s/2^d)
  if (tid < 2) {
    const int Q = tid == 0 ? P.Qy : P.Qx;
    const int o = tid == 0 ? i0 : j0;
    int s = (o << K) - Q - 1;
    for (int l = m - 1; l >= 0; --l) {
      s >>= 1;
      sR[tid][0][l] = s;
    }
  }
  if (tid == 0) {  // window side of level l = m-d: P(d) = P(d-1)/2 + 1, P(0) = FW (O(m), incremental)
    int off = 0, p = G::FW;
    for (int l = m - 1; l >= 0; --l) {
      p = p / 2 + 1;
      sDoff[l] = off;
      off += (l == m - 1) ? 3 * (p + 1) * G::WS1 : 3 * (p + 1) * (p + 1);
      sR[0][1][l] = p;
      sR[1][1][l] = p;
    }
    sDoff[m] = off;
  }
  __syncthreads();

  HS_PHASE(1)
  // ---- detail windows in two cp.async groups: group A = ancestors' windows (levels <= m-3),
  //      group B = the large windows of levels m-2 and m-1; the ancestors' top-down runs while
  //      group B is still in flight.  Per level d = m - l the window side is a compile-time
  //      constant, so the element decode uses constant divisors.
  load_windows<G, 3, K>(in, sDet, sR, sDoff, m);             // group A: d = 3 .. K (levels c .. m-3)
  cp_async_commit();
  if (m - 1 >= 2)
    load_window_vec<G>(in, sDet, sR, sDoff, m);               // group B: d = 1 (16-byte chunks)
  else
    load_windows<G, 1, 1>(in, sDet, sR, sDoff, m);
  load_windows<G, 2, 2>(in, sDet, sR, sDoff, m);             // group B: d = 2
  cp_async_commit();
  if (c > 0) {  // unshifted level-c fields (fp64, coarse_fields_kernel) -> FT, while the copies fly
    const int gc = 1 << c, cm = gc - 1;
    const int pw = sR[0][1][c], ys = sR[0][0][c], xs = sR[1][0][c];
    const double* src = reinterpret_cast<const double*>(reinterpret_cast<const char*>(args.ws) +
                                                        (long long)g * args.ws_face_stride + 3ll * gc * gc * 8);
    FT* dst = sCh + ((((K - 2) & 1) == 0) ? 3 * G::ANC_MAX * G::ANC_MAX : 0);
    for (int e = tid; e < 3 * pw * pw; e += kThreads) {
      const int t = e / (pw * pw), rem = e - t * pw * pw;
      const int a = rem / pw, bb = rem - a * pw;
      dst[t * G::ANC_MAX * G::ANC_MAX + a * pw + bb] =
          FT(__ldcg(src + (long long)t * gc * gc + (long long)((ys + a) & cm) * gc + ((xs + bb) & cm)));
    }
  }
  cp_async_wait_group1();                                    // A complete, B may be in flight
  __syncthreads();

  HS_PHASE(2)
  // ---- (1) ancestors top-down: fields of levels 1 .. m-1 (level m-1 -> sB1, others alias sCh)
  auto ancestor_level = [&](int l) {
    const int pw = sR[0][1][l];
    const int ys = sR[0][0][l], xs = sR[1][0][l];
    const int dw = pw + 1, dplane = dw * dw;
    const float* dt = sDet + sDoff[l];
    const FT asc = FT(pow2f(l));
    const bool to_b1 = (l + 1 == m - 1);
    // children at level l+1 land in: level m-1 -> sB1 (side CB); else alternate halves of sCh
    FT* cf = to_b1 ? sB1 : sCh + ((((m - 2 - l) & 1) == 0) ? 0 : 3 * G::ANC_MAX * G::ANC_MAX);
    const int cside = 2 * pw;
    const int cplane = to_b1 ? CB * CB : G::ANC_MAX * G::ANC_MAX;
    const FT* pf = sCh + ((((m - 2 - l) & 1) == 0) ? 3 * G::ANC_MAX * G::ANC_MAX : 0);
    const int pplane = G::ANC_MAX * G::ANC_MAX;
    int pstride = 0, poy = 0, pox = 0;
    if (l == c) {
      pstride = pw;                 // the level-c window loaded from coarse_fields_kernel
    } else if (l > 0) {
      pstride = 2 * sR[0][1][l - 1];
      poy = ys - 2 * sR[0][0][l - 1];
      pox = xs - 2 * sR[1][0][l - 1];
    }
    const float inv_pw = inv_small(pw);
    for (int idx = tid; idx < pw * pw; idx += kThreads) {
      const int pi = div_small(idx, inv_pw), pj = idx - pi * pw;
      FT dd[2][2][2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int o = (pi + u) * dw + (pj + v);
          const FT H = FT(dt[o]) * asc, V = FT(dt[dplane + o]) * asc, D = FT(dt[2 * dplane + o]) * asc;
          dd[u][v][0][0] = H + V + D;
          dd[u][v][0][1] = -H + V - D;
          dd[u][v][1][0] = H - V - D;
          dd[u][v][1][1] = -H - V + D;
        }
      FT Xl = FT(0), Yl = FT(0), Zl = FT(0);
      if (l > 0) {
        const int po = (pi + poy) * pstride + (pj + pox);
        Xl = pf[po];
        Yl = pf[pplane + po];
        Zl = pf[2 * pplane + po];
      }
      const int co = (2 * pi) * cside + 2 * pj;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        cf[co + a * cside + 0] = dd[0][0][a][0] - dd[0][0][a][1];
        cf[co + a * cside + 1] = Xl + dd[0][0][a][1] - dd[0][1][a][0];
      }
#pragma unroll
      for (int bq = 0; bq < 2; ++bq) {
        cf[cplane + co + bq] = dd[0][0][0][bq] - dd[0][0][1][bq];
        cf[cplane + co + cside + bq] = Yl + dd[0][0][1][bq] - dd[1][0][0][bq];
      }
      cf[2 * cplane + co] = dd[0][0][0][0] - dd[0][0][0][1] - dd[0][0][1][0] + dd[0][0][1][1];
      cf[2 * cplane + co + 1] = dd[0][0][0][1] - dd[0][0][1][1] - dd[0][1][0][0] + dd[0][1][1][0];
      cf[2 * cplane + co + cside] = dd[0][0][1][0] - dd[0][0][1][1] - dd[1][0][0][0] + dd[1][0][0][1];
      cf[2 * cplane + co + cside + 1] =
          Zl + dd[0][0][1][1] - dd[0][1][1][0] - dd[1][0][0][1] + dd[1][1][0][0];
    }
    __syncthreads();
  };
  HS_PHASE(3)
  for (int l = c; l + 2 < m; ++l) ancestor_level(l);  // uses group A only
  cp_async_wait_all();
  __syncthreads();
  HS_PHASE(4)
  if (m >= 2) ancestor_level(m - 2);                  // level m-1 fields (group B)

  HS_PHASE(5)
  // ---- per field t in {X, Y, Z}: (1') its level-m children (one parity-split plane, so three
  //      fields never share memory) then (2)+(3) the fused shift + first bottom-up stencil with a
  //      register-sliding window down each thread's strip; shifted level-(m-1) field t -> sB1
  //      plane t (whose unshifted content only field t's children needed), outputs -> global
  {
    const int l = m - 1;
    const int ys = sR[0][0][l], xs = sR[1][0][l];
    constexpr int DW = G::P1 + 1;
    const bool vec = (m - 1 >= 2);                 // level m-1 window stored with padded rows
    const int RW = vec ? G::WS1 : DW;              // row stride
    const int DPL = DW * RW;                       // plane stride
    const float* dt = sDet + sDoff[l] + (vec ? (sR[1][0][l] & 3) : 0);
    const FT asc = FT(pow2f(l));
    int poy = 0, pox = 0;
    if (l > 0) {
      poy = ys - 2 * sR[0][0][l - 1];
      pox = xs - 2 * sR[1][0][l - 1];
    }
    constexpr int NP = G::P1 * G::P1;

    const int k1 = K - 1;
    const int Ssy = i0 << k1, Ssx = j0 << k1;
    constexpr int ON1 = TC << (K - 1);
    const int Cy = 2 * sR[0][0][m - 1], Cx = 2 * sR[1][0][m - 1];
    const FT wy1 = FT(P.wy), wx1 = FT(P.wx);
    const FT wy0 = FT(1) - wy1, wx0 = FT(1) - wx1;
    const FT ta = wx1, tb0 = wx0 + FT(2) * wx1, tb1 = FT(2) * wx0 + wx1, tcc = wx0;
    const FT ua = wy1, ub0 = wy0 + FT(2) * wy1, ub1 = FT(2) * wy0 + wy1, uc = wy0;
    const FT q = FT(0.25);
    const int gl = 1 << l;
    const FT osc = FT(pow2f(-l));
    const bool emit = l < band;
    const int strip = tid / SN1, jj = tid - strip * SN1;

#pragma unroll
    for (int fld = 0; fld < 3; ++fld) {
      // (1') children of field fld
#pragma unroll 1
      for (int idx = tid; idx < NP; idx += kThreads) {
        const int pi = idx / G::P1, pj = idx - pi * G::P1;  // constant divisor
        const int o = pi * RW + pj;
        const FT H0 = FT(dt[o]) * asc, V0 = FT(dt[DPL + o]) * asc, D0 = FT(dt[2 * DPL + o]) * asc;
        const FT d00 = H0 + V0 + D0, d01 = -H0 + V0 - D0, d10 = H0 - V0 - D0, d11 = -H0 - V0 + D0;
        FT pf = FT(0);
        if (l > 0) pf = sB1[fld * CB * CB + (pi + poy) * CB + (pj + pox)];
        FT* c0 = sCh + (2 * pi) * HC + pj;  // even plane, row 2pi
        if (fld == 0) {
          const int o1 = o + 1;
          const FT H1 = FT(dt[o1]) * asc, V1 = FT(dt[DPL + o1]) * asc, D1 = FT(dt[2 * DPL + o1]) * asc;
          const FT r00 = H1 + V1 + D1, r10 = H1 - V1 - D1;
          c0[0] = d00 - d01;
          c0[PLANE_C] = pf + d01 - r00;
          c0[HC] = d10 - d11;
          c0[PLANE_C + HC] = pf + d11 - r10;
        } else if (fld == 1) {
          const int o2 = o + RW;
          const FT H2 = FT(dt[o2]) * asc, V2 = FT(dt[DPL + o2]) * asc, D2 = FT(dt[2 * DPL + o2]) * asc;
          const FT b00 = H2 + V2 + D2, b01 = -H2 + V2 - D2;
          c0[0] = d00 - d10;
          c0[PLANE_C] = d01 - d11;
          c0[HC] = pf + d10 - b00;
          c0[PLANE_C + HC] = pf + d11 - b01;
        } else {
          const int o1 = o + 1, o2 = o + RW, o3 = o + RW + 1;
          const FT H1 = FT(dt[o1]) * asc, V1 = FT(dt[DPL + o1]) * asc, D1 = FT(dt[2 * DPL + o1]) * asc;
          const FT H2 = FT(dt[o2]) * asc, V2 = FT(dt[DPL + o2]) * asc, D2 = FT(dt[2 * DPL + o2]) * asc;
          const FT H3 = FT(dt[o3]) * asc, V3 = FT(dt[DPL + o3]) * asc, D3 = FT(dt[2 * DPL + o3]) * asc;
          const FT r00 = H1 + V1 + D1, r10 = H1 - V1 - D1;
          const FT b00 = H2 + V2 + D2, b01 = -H2 + V2 - D2;
          const FT g00 = H3 + V3 + D3;
          c0[0] = FT(4) * D0;
          c0[PLANE_C] = d01 - d11 - r00 + r10;
          c0[HC] = d10 - d11 - b00 + b01;
          c0[PLANE_C + HC] = pf + d11 - r10 - b01 + g00;
        }
      }
      __syncthreads();

      // (2)+(3) fused stencil of field fld
      if (strip < G::NSTRIP) {
        const int ii0 = strip * G::RSS;
        const int rb = 2 * (Ssy + ii0) - P.Qy - Cy - 1;  // window row 0 = tap -1 of row ii0
        constexpr int NW = 2 * G::RSS + 2;
        const FT* base[4];
#pragma unroll
        for (int vv = 0; vv < 4; ++vv) {
          const int cl = 2 * (Ssx + jj) - P.Qx - Cx + vv - 1;
          base[vv] = sCh + (cl & 1) * PLANE_C + rb * HC + (cl >> 1);
        }
        FT hA[NW], hB[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const FT x_1 = base[0][w * HC], x0 = base[1][w * HC], x1 = base[2][w * HC];
          if (fld == 1) {
            hA[w] = wx1 * x_1 + x0 + wx0 * x1;
            hB[w] = hA[w];
          } else {
            const FT x2 = base[3][w * HC];
            hA[w] = ta * x_1 + tb0 * x0 + tb1 * x1 + tcc * x2;
            hB[w] = wx1 * x_1 + wx0 * x0;
          }
        }
        FT* dstS = sB1 + fld * CB * CB + ii0 * SN1 + jj;
        float* ob = out + (long long)gl * gl * (1 + fld) + (Ssy + ii0) * gl + (Ssx + jj);
        const bool emit_col = emit && jj < ON1;
#pragma unroll
        for (int r = 0; r < G::RSS; ++r) {
          const int ii = ii0 + r;
          if (ii < SN1) {
            const int u = 2 * r;
            FT fv, dv;
            if (fld == 0) {
              fv = q * (wy1 * hA[u] + hA[u + 1] + wy0 * hA[u + 2]);
              dv = q * (wy1 * hB[u] + hB[u + 1] + wy0 * hB[u + 2]);
            } else {
              fv = q * (ua * hA[u] + ub0 * hA[u + 1] + ub1 * hA[u + 2] + uc * hA[u + 3]);
              dv = q * (wy1 * hB[u] + wy0 * hB[u + 1]);
            }
            dstS[r * SN1] = fv;
            if (emit_col && ii < ON1) ob[r * gl] = (float)(dv * osc);
          }
        }
      }
      __syncthreads();
      if (fld == 0) { HS_PHASE(6) }
    }
  }

  HS_PHASE(7)
  // ---- (3) plain bottom-up for levels m-2 .. c (compile-time windows), sB1 <-> sCh
  const FT* srcS = sB1;
  int srcN = SN1, srcPlane = CB * CB;
  const FT q = FT(0.25);
#pragma unroll
  for (int e = K - 2; e >= 0; --e) {
    const int lev = c + e;
    const int Sn = G::SN(e);
    const int On = TC << e;
    const int Ssy = i0 << e, Ssx = j0 << e;
    FT* dst = ((K - 2 - e) & 1) == 0 ? sCh : sB1;
    const int dstPlane = ((K - 2 - e) & 1) == 0 ? Sn * Sn : CB * CB;
    const int gl = 1 << lev;
    const FT osc = FT(pow2f(-lev));
    const bool emit = lev < band;
    const float inv_sn = inv_small(Sn);
    for (int idx = tid; idx < Sn * Sn; idx += kThreads) {
      const int ii = div_small(idx, inv_sn), jj = idx - ii * Sn;
      const int a2 = 2 * ii, b2 = 2 * jj;
      const FT* X = srcS + a2 * srcN + b2;
      const FT* Y = srcS + srcPlane + a2 * srcN + b2;
      const FT* Z = srcS + 2 * srcPlane + a2 * srcN + b2;
      const FT Xn = q * (X[0] + FT(2) * X[1] + X[2] + X[srcN] + FT(2) * X[srcN + 1] + X[srcN + 2]);
      const FT Yn = q * (Y[0] + FT(2) * Y[srcN] + Y[2 * srcN] + Y[1] + FT(2) * Y[srcN + 1] + Y[2 * srcN + 1]);
      const FT Zn = q * ((Z[0] + FT(2) * Z[1] + Z[2]) + FT(2) * (Z[srcN] + FT(2) * Z[srcN + 1] + Z[srcN + 2]) +
                         (Z[2 * srcN] + FT(2) * Z[2 * srcN + 1] + Z[2 * srcN + 2]));
      dst[ii * Sn + jj] = Xn;
      dst[dstPlane + ii * Sn + jj] = Yn;
      dst[2 * dstPlane + ii * Sn + jj] = Zn;
      if (ii < On && jj < On && emit) {
        const int o = (Ssy + ii) * gl + (Ssx + jj);
        out[(long long)gl * gl * 1 + o] = (float)(q * (X[0] + X[srcN]) * osc);
        out[(long long)gl * gl * 2 + o] = (float)(q * (Y[0] + Y[1]) * osc);
        out[(long long)gl * gl * 3 + o] = (float)(q * Z[0] * osc);
      }
    }
    __syncthreads();
    srcS = dst;
    srcN = Sn;
    srcPlane = dstPlane;
  }
  // srcS holds the shifted level-c fields over the owned tile (srcN = TC when K >= 2; SN1 = TC when K = 1)

  HS_PHASE(8)
  if (blockIdx.x == 0 && tid == 0) out[0] = __ldg(in);  // scaling coefficient: unchanged (R8)
  if (c == 0) return;

  // ---- publish the owned shifted level-c fields (coarse_finish_kernel runs the bottom-up c -> 0)
  const int gc = 1 << c;
  FT* wsf = reinterpret_cast<FT*>(reinterpret_cast<char*>(args.ws) + (long long)g * args.ws_face_stride);
  for (int idx = tid; idx < 3 * TC * TC; idx += kThreads) {
    const int fld = idx / (TC * TC), r = idx - fld * TC * TC;
    const int ii = r / TC, jj = r - ii * TC;
    wsf[(long long)fld * gc * gc + (long long)(i0 + ii) * gc + (j0 + jj)] = srcS[fld * srcPlane + ii * srcN + jj];
  }
  HS_PHASE(9)
}

// (1) over the full grid of one face up to the tile-root level c: the unshifted level-c fields.
// Intermediate levels ping-pong in shared memory when they fit (else through the not yet used
// shifted-field and scratch areas of the workspace).
constexpr int kFieldsSmem = 48 * 1024;
__global__ void __launch_bounds__(kThreads) coarse_fields_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char fsmem[];
  const int g = blockIdx.x;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int c = P.m > KF ? P.m - KF : 0;
  if (c == 0 || (args.band_path && band_level(P.m))) return;   // band faces: shift2d_band_kernel
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in = args.in + (long long)b * args.in_batch_stride + (long long)f * args.in_face_stride;
  using FT = double;   // always fp64: the coarse recursion carries pixel-value-scale errors otherwise
  FT* wsf = reinterpret_cast<FT*>(reinterpret_cast<char*>(args.ws) + (long long)g * args.ws_face_stride);
  const long long GC = 1ll << (2 * c);
  const bool in_smem = (15ll * (GC / 16)) * (long long)sizeof(FT) <= kFieldsSmem;   // 3 (4^(c-1) + 4^(c-2))
  FT* const bufA = in_smem ? reinterpret_cast<FT*>(fsmem) + 3 * (GC / 4) : wsf;        // level c-2, c-4, ...
  FT* const bufB = in_smem ? reinterpret_cast<FT*>(fsmem) : wsf + 6 * GC;             // level c-1, c-3, ...
  FT* const fin = wsf + 3 * GC;         // unshifted level-c fields
  for (int l = 0; l < c; ++l) {
    const int gl = 1 << l, G2 = 2 * gl;
    const FT asc = FT(pow2f(l));
    const FT* cur = ((c - l) & 1) ? bufB : bufA;       // level l fields (l > 0)
    FT* nxt = (l + 1 == c) ? fin : (((c - l - 1) & 1) ? bufB : bufA);
    for (int idx = threadIdx.x; idx < gl * gl; idx += blockDim.x) {
      const int i = idx >> l, j = idx & (gl - 1);
      FT d[2][2][2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const long long o = (long long)((i + u) & (gl - 1)) * gl + ((j + v) & (gl - 1));
          const FT H = FT(__ldg(in + (long long)gl * gl * 1 + o)) * asc;
          const FT V = FT(__ldg(in + (long long)gl * gl * 2 + o)) * asc;
          const FT D = FT(__ldg(in + (long long)gl * gl * 3 + o)) * asc;
          d[u][v][0][0] = H + V + D;
          d[u][v][0][1] = -H + V - D;
          d[u][v][1][0] = H - V - D;
          d[u][v][1][1] = -H - V + D;
        }
      FT Xl = FT(0), Yl = FT(0), Zl = FT(0);
      if (l > 0) {
        if (in_smem) {
          Xl = cur[idx];
          Yl = cur[gl * gl + idx];
          Zl = cur[2 * gl * gl + idx];
        } else {
          Xl = __ldcg(cur + idx);
          Yl = __ldcg(cur + gl * gl + idx);
          Zl = __ldcg(cur + 2 * gl * gl + idx);
        }
      }
      FT cx[2][2], cy[2][2], cz[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        cx[a][0] = d[0][0][a][0] - d[0][0][a][1];
        cx[a][1] = Xl + d[0][0][a][1] - d[0][1][a][0];
      }
#pragma unroll
      for (int bq = 0; bq < 2; ++bq) {
        cy[0][bq] = d[0][0][0][bq] - d[0][0][1][bq];
        cy[1][bq] = Yl + d[0][0][1][bq] - d[1][0][0][bq];
      }
      cz[0][0] = d[0][0][0][0] - d[0][0][0][1] - d[0][0][1][0] + d[0][0][1][1];
      cz[0][1] = d[0][0][0][1] - d[0][0][1][1] - d[0][1][0][0] + d[0][1][1][0];
      cz[1][0] = d[0][0][1][0] - d[0][0][1][1] - d[1][0][0][0] + d[1][0][0][1];
      cz[1][1] = Zl + d[0][0][1][1] - d[0][1][1][0] - d[1][0][0][1] + d[1][1][0][0];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bq = 0; bq < 2; ++bq) {
          const long long o = (long long)(2 * i + a) * G2 + (2 * j + bq);
          nxt[o] = cx[a][bq];
          nxt[(long long)G2 * G2 + o] = cy[a][bq];
          nxt[2ll * G2 * G2 + o] = cz[a][bq];
        }
    }
    __syncthreads();
  }
}

// The coarse bottom-up c -> 0 of one face from the tiles' shifted level-c fields.
constexpr int kFinishSmem = 64 * 1024;
template <typename FT>
__global__ void __launch_bounds__(kThreads) coarse_finish_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int g = blockIdx.x;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int c = P.m > KF ? P.m - KF : 0;
  if (c == 0 || (args.band_path && band_level(P.m))) return;   // band faces: band_finish_kernel
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  char* wsb = reinterpret_cast<char*>(args.ws) + (long long)g * args.ws_face_stride;
  FT* wsf = reinterpret_cast<FT*>(wsb);
  const int gc = 1 << c;
  const long long need = 3ll * gc * gc + 3ll * (gc / 2) * (gc / 2);
  if (need * (long long)sizeof(FT) <= (long long)kFinishSmem) {
    FT* A = reinterpret_cast<FT*>(smem);
    FT* B0 = A + 3 * gc * gc;
    for (int idx = threadIdx.x; idx < 3 * gc * gc; idx += kThreads) A[idx] = __ldcg(wsf + idx);
    __syncthreads();
    coarse_finish<FT>(A, B0, A, c, out, args.band, false);
  } else {
    coarse_finish<FT>(wsf, reinterpret_cast<FT*>(wsb + 6ll * gc * gc * 8), wsf, c, out, args.band, true);
  }
}

template <typename FT>
constexpr int max_tile_smem() {
  const int v[6] = {TSmem<FT, 3, 8>::BYTES, TSmem<FT, 3, 4>::BYTES, TSmem<FT, 3, 2>::BYTES,
                    TSmem<FT, 3, 1>::BYTES, TSmem<FT, 2, 1>::BYTES, TSmem<FT, 1, 1>::BYTES};
  int mx = 0;
  for (int x : v) mx = x > mx ? x : mx;
  return mx;
}

template <typename FT>
__global__ void __launch_bounds__(kThreads, sizeof(FT) == 4 ? 3 : 2) shift2d_tile_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sR[2][2][HS_MAX_LOG2N + 1];
  __shared__ int sDoff[HS_MAX_LOG2N + 2];
  const int g = blockIdx.y;  // face within this launch
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int m = P.m;
  if (m == 0) return;  // identity: handled by permute_kernel
  if (args.band_path && band_level(m)) return;   // shift2d_band_kernel
  const int c = m > KF ? m - KF : 0;
  const int k = m - c;
  const int tc = (1 << c) < TC ? (1 << c) : TC;
  const int tpr = (1 << c) / tc;
  if ((int)blockIdx.x >= tpr * tpr) return;
  const int i0 = (blockIdx.x / tpr) * tc;
  const int j0 = (blockIdx.x % tpr) * tc;
  if (k == 3) {
    switch (tc) {
      case 8: tile_body<FT, 3, 8>(args, smem, P, g, m, c, i0, j0, sR, sDoff); break;
      case 4: tile_body<FT, 3, 4>(args, smem, P, g, m, c, i0, j0, sR, sDoff); break;
      case 2: tile_body<FT, 3, 2>(args, smem, P, g, m, c, i0, j0, sR, sDoff); break;
      default: tile_body<FT, 3, 1>(args, smem, P, g, m, c, i0, j0, sR, sDoff); break;
    }
  } else if (k == 2) {
    tile_body<FT, 2, 1>(args, smem, P, g, m, c, i0, j0, sR, sDoff);
  } else {
    tile_body<FT, 1, 1>(args, smem, P, g, m, c, i0, j0, sR, sDoff);
  }
}

// Levels >= m of faces with a dyadic shift are exact circular permutations; the
// scaling coefficient of identity faces (m = 0) is copied here too.
__global__ void permute_kernel(const __grid_constant__ ShiftArgs args) {
  const int g = blockIdx.y;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int n = args.log2n;
  const int m = P.m;
  if (m >= args.band && m != 0) return;
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in =
      args.in + (long long)b * args.in_batch_stride + (long long)f * args.in_face_stride;
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  const long long lo = (m == 0) ? 0 : (1ll << (2 * m));
  const long long hi = 1ll << (2 * args.band);
  for (long long idx = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < hi;
       idx += (long long)gridDim.x * blockDim.x) {
    if (idx == 0) {
      out[0] = in[0];
      continue;
    }
    const int l = (63 - __clzll(idx)) >> 1;  // 4^l <= idx < 4^(l+1)
    const long long base = 1ll << (2 * l);
    const long long r = idx - base;
    const int t = (int)(r >> (2 * l));
    const long long cell = r & (base - 1);
    const int i = (int)(cell >> l), j = (int)(cell & ((1 << l) - 1));
    const int sh = n - l;
    const int si = (i - (P.qy >> sh)) & ((1 << l) - 1);
    const int sj = (j - (P.qx >> sh)) & ((1 << l) - 1);
    out[idx] = __ldg(in + base * (1 + t) + ((long long)si << l) + sj);
  }
}

template <typename FT>
hs_status launch_tiles(ShiftArgs& a, int max_tiles, bool any_coarse, bool any_tile, int max_band_m, cudaStream_t st) {
  HS_SMEM_ATTR(shift2d_tile_kernel<FT>, max_tile_smem<FT>());
  HS_SMEM_ATTR(coarse_fields_kernel, kFieldsSmem);
  HS_SMEM_ATTR(coarse_finish_kernel<FT>, kFinishSmem);
  if (any_coarse) {
    coarse_fields_kernel<<<a.num_faces, kThreads, kFieldsSmem, st>>>(a);
    HS_CHECK_LAUNCH("coarse_fields_kernel");
  }
  if (any_tile) {
    shift2d_tile_kernel<FT><<<dim3(max_tiles, a.num_faces), kThreads, max_tile_smem<FT>(), st>>>(a);
    HS_CHECK_LAUNCH("shift2d_tile_kernel");
  }
  if (max_band_m > 0) {
    hs_status s = launch_shift2d_band(a, max_band_m, st);
    if (s != HS_OK) return s;
  }
  if (any_coarse) {
    coarse_finish_kernel<FT><<<a.num_faces, kThreads, kFinishSmem, st>>>(a);
    HS_CHECK_LAUNCH("coarse_finish_kernel");
  }
  return HS_OK;
}

// Small faces (N <= 32): the whole shift of one face in one CTA -- the pyramid is read once into
// shared memory (one global round trip instead of one per phase of the tile path), then the
// top-down to the working level m, the shift at m, the bottom-up m -> 0 (coarse_finish) and the
// permuted levels >= m, all in fp64 shared memory.  One launch per call.
constexpr int kSmallMaxLog2n = 5;
constexpr int kSmallSmem = (1 << (2 * kSmallMaxLog2n)) * 4 +                           // the pyramid
                           (3 * (1 << (2 * kSmallMaxLog2n)) * 2 + 3 * (1 << (2 * (kSmallMaxLog2n - 1)))) * 8;

__global__ void __launch_bounds__(kThreads) shift2d_small_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) unsigned char ssm[];
  const int g = blockIdx.x;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int n = args.log2n, m = P.m, band = args.band;
  const int NN = 1 << (2 * n);
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in = args.in + (long long)b * args.in_batch_stride + (long long)f * args.in_face_stride;
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  float* C = reinterpret_cast<float*>(ssm);                       // the input pyramid
  double* FA = reinterpret_cast<double*>(ssm + (size_t)NN * 4);   // 3 x 4^m
  double* FB = FA + 3 * (1 << (2 * m));                           // 3 x 4^m
  double* FC = FB + 3 * (1 << (2 * m));                           // 3 x 4^(m-1) (bottom-up scratch)
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) C[idx] = __ldg(in + idx);
  __syncthreads();
  // levels >= m (up to the band): exact permutations; the scaling coefficient is shift invariant
  const int hi = 1 << (2 * band);
  for (int idx = threadIdx.x; idx < hi; idx += blockDim.x) {
    if (idx == 0) {
      out[0] = C[0];
      continue;
    }
    const int l = (31 - __clz(idx)) >> 1;
    if (l < m) continue;
    const int base = 1 << (2 * l), r = idx - base, t = r >> (2 * l), cell = r & (base - 1);
    const int i = cell >> l, j = cell & ((1 << l) - 1), sh = n - l;
    const int si = (i - (P.qy >> sh)) & ((1 << l) - 1), sj = (j - (P.qx >> sh)) & ((1 << l) - 1);
    out[idx] = C[base * (1 + t) + (si << l) + sj];
  }
  if (m == 0) return;
  // top-down: fields of levels 1 .. m (X, Y, Z), ping-pong FA / FB, level m ends in FA
  for (int l = 0; l < m; ++l) {
    const int gl = 1 << l, G2 = 2 * gl;
    const double asc = (double)pow2f(l);
    const double* cur = ((m - l) & 1) ? FB : FA;
    double* nxt = ((m - l - 1) & 1) ? FB : FA;
    for (int idx = threadIdx.x; idx < gl * gl; idx += blockDim.x) {
      const int i = idx >> l, j = idx & (gl - 1);
      double d[2][2][2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int o = ((i + u) & (gl - 1)) * gl + ((j + v) & (gl - 1));
          const double H = (double)C[gl * gl * 1 + o] * asc;
          const double V = (double)C[gl * gl * 2 + o] * asc;
          const double D = (double)C[gl * gl * 3 + o] * asc;
          d[u][v][0][0] = H + V + D;
          d[u][v][0][1] = -H + V - D;
          d[u][v][1][0] = H - V - D;
          d[u][v][1][1] = -H - V + D;
        }
      double Xl = 0.0, Yl = 0.0, Zl = 0.0;
      if (l > 0) {
        Xl = cur[idx];
        Yl = cur[gl * gl + idx];
        Zl = cur[2 * gl * gl + idx];
      }
      double cx[2][2], cy[2][2], cz[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        cx[a][0] = d[0][0][a][0] - d[0][0][a][1];
        cx[a][1] = Xl + d[0][0][a][1] - d[0][1][a][0];
      }
#pragma unroll
      for (int bq = 0; bq < 2; ++bq) {
        cy[0][bq] = d[0][0][0][bq] - d[0][0][1][bq];
        cy[1][bq] = Yl + d[0][0][1][bq] - d[1][0][0][bq];
      }
      cz[0][0] = d[0][0][0][0] - d[0][0][0][1] - d[0][0][1][0] + d[0][0][1][1];
      cz[0][1] = d[0][0][0][1] - d[0][0][1][1] - d[0][1][0][0] + d[0][1][1][0];
      cz[1][0] = d[0][0][1][0] - d[0][0][1][1] - d[1][0][0][0] + d[1][0][0][1];
      cz[1][1] = Zl + d[0][0][1][1] - d[0][1][1][0] - d[1][0][0][1] + d[1][1][0][0];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bq = 0; bq < 2; ++bq) {
          const int o = (2 * i + a) * G2 + (2 * j + bq);
          nxt[o] = cx[a][bq];
          nxt[G2 * G2 + o] = cy[a][bq];
          nxt[2 * G2 * G2 + o] = cz[a][bq];
        }
    }
    __syncthreads();
  }
  // the shift at level m: box projection with weights (1 - phi, phi) on offsets Q, Q + 1
  const int gm = 1 << m, GM = gm * gm;
  const double wy1 = (double)P.wy, wx1 = (double)P.wx, wy0 = 1.0 - wy1, wx0 = 1.0 - wx1;
  for (int idx = threadIdx.x; idx < 3 * GM; idx += blockDim.x) {
    const int fl = idx / GM, cell = idx - fl * GM, y = cell >> m, x = cell & (gm - 1);
    const double* F = FA + fl * GM;
    const int y0 = (y - P.Qy) & (gm - 1), y1 = (y - P.Qy - 1) & (gm - 1);
    const int x0 = (x - P.Qx) & (gm - 1), x1 = (x - P.Qx - 1) & (gm - 1);
    FB[idx] = wy0 * (wx0 * F[y0 * gm + x0] + wx1 * F[y0 * gm + x1]) + wy1 * (wx0 * F[y1 * gm + x0] + wx1 * F[y1 * gm + x1]);
  }
  __syncthreads();
  // bottom-up m -> 0 (details of levels < band)
  coarse_finish<double>(FB, FC, FA, m, out, band, false);
}

}  // namespace

hs_status launch_shift2d(ShiftArgs& a, int max_tiles, bool any_coarse, bool any_perm, bool any_tile, int max_band_m,
                         cudaStream_t st) {
  if (a.log2n <= kSmallMaxLog2n) {
    const size_t smem = (size_t)(1 << (2 * a.log2n)) * 4 +
                        ((size_t)3 * (1 << (2 * a.log2n)) * 2 + 3 * (1 << (2 * (a.log2n > 0 ? a.log2n - 1 : 0)))) * 8;
    HS_SMEM_ATTR(shift2d_small_kernel, kSmallSmem);
    shift2d_small_kernel<<<a.num_faces, kThreads, smem, st>>>(a);
    HS_CHECK_LAUNCH("shift2d_small_kernel");
    return HS_OK;
  }
  if (max_tiles > 0) {
    // fp64 fields at every size: fp32 rounding in the difference fields is amplified ~2^(n-l) on a
    // band of level l; the randomised sweep (tests/test_gpu_fuzz.py) measured
    // 2e-5 for white noise at N = 64 with fp32 fields.
    hs_status s = launch_tiles<double>(a, max_tiles, any_coarse, any_tile, a.band_path ? max_band_m : 0, st);
    if (s != HS_OK) return s;
  }
  if (any_perm) {
    long long span = 1ll << (2 * a.band);
    int blocks = (int)((span + 255) / 256);
    if (blocks > 64) blocks = 64;
    if (blocks < 1) blocks = 1;
    permute_kernel<<<dim3(blocks, a.num_faces), 256, 0, st>>>(a);
    HS_CHECK_LAUNCH("permute_kernel");
  }
  return HS_OK;
}

int shift2d_tiles_for(int m) {
  if (m == 0) return 0;
  const int c = coarse_level(m);
  const int tc = (1 << c) < kTileTC ? (1 << c) : kTileTC;
  const int tpr = (1 << c) / tc;
  return tpr * tpr;
}

}  // namespace hs
