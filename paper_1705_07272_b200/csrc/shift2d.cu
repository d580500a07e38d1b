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
// Tiling: a CTA owns a TC x TC tile at the tile-root level c = max(0, m - KF) and every output
// coefficient below it at levels c..m-1.  All detail windows it needs (its ancestors' few cells
// at levels < c plus tile + halo at levels c..m-1) are fetched up front with cp.async (one
// latency round trip); it then recomputes the ancestors' fields top-down from level 0, runs
// (1)-(3) over its window (all periodic index arithmetic on unwrapped coordinates), writes its
// outputs and its shifted level-c fields.  The last CTA of a face to finish (atomic ticket) runs
// the coarse bottom-up c -> 0.  Levels >= m (dyadic shifts) are exact permutations.
//
// Field precision FT: fp32 for log2n <= 8; fp64 above (DESIGN.md §4.1 error model: fine-level
// fp32 rounding is amplified ~2^(n-l) on the coarse outputs of large faces).
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

constexpr int KF = kTileKF;
constexpr int TC = kTileTC;
constexpr int kThreads = 256;
// compile-time maxima of the per-axis region sizes
constexpr int PM1 = (1 << (KF - 1)) * (TC + 1) + 1;   // parents at level m-1          (37)
constexpr int PM2 = (1 << (KF - 2)) * (TC + 1) + 1;   // parents at level m-2          (19)
constexpr int CB = 2 * PM2;                            // level m-1 field plane side    (38)
constexpr int CSM = PM2 + 1;                           // level <= m-2 field plane side (20)
constexpr int CM = 2 * PM1;                            // level m children plane side   (74)
constexpr int SM1 = (1 << (KF - 1)) * (TC + 1) - 1;   // shifted window at m-1         (35)
constexpr int SM2 = (1 << (KF - 2)) * (TC + 1) - 1;   // shifted window at m-2         (17)
constexpr int DET_FLOATS = 6336;                       // all detail windows, <= 12 levels
static_assert(SM1 <= CB && SM2 <= CSM && PM1 <= CB, "aliasing assumptions");

template <typename FT>
struct Smem {
  static constexpr int DET = 0;                                        // float[DET_FLOATS]
  static constexpr int FB = DET + DET_FLOATS * 4;                       // FT[3][CB*CB]
  static constexpr int FS = FB + 3 * CB * CB * (int)sizeof(FT);         // FT[3][CSM*CSM]
  static constexpr int BIG = FS + 3 * CSM * CSM * (int)sizeof(FT);      // FT[CM*CM]
  static constexpr int BYTES = BIG + CM * CM * (int)sizeof(FT);
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Exact 2^e for |e| < 127 (no libm call).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// floor(x / n) for 0 <= x < 2^16, 1 <= n < 2^10 from an approximate reciprocal: (x + 1/2)/n is at
// least 1/(2n) away from an integer and the float error is < 2^-21 * 2^16 / n, so the floor is exact.
__device__ __forceinline__ int div_small(int x, float inv_n) { return __float2int_rd(((float)x + 0.5f) * inv_n); }
__device__ __forceinline__ float inv_small(int n) { return __fdividef(1.0f, (float)n); }

// Block-stride walk over a rows x cols grid (flat index idx = r * cols + c) without an integer
// division: one reciprocal division at the start, then incremental row/column updates.
struct Walk2 {
  int idx, r, c, dr, dc, cols;
  __device__ __forceinline__ Walk2(int total, int ncols) : cols(ncols) {
    const float inv = inv_small(ncols);
    idx = threadIdx.x;
    r = div_small(idx, inv);
    c = idx - r * cols;
    dr = div_small(blockDim.x, inv);
    dc = blockDim.x - dr * cols;
    (void)total;
  }
  __device__ __forceinline__ void next() {
    idx += blockDim.x;
    r += dr;
    c += dc;
    if (c >= cols) {
      c -= cols;
      ++r;
    }
  }
};

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

template <typename FT>
__global__ void __launch_bounds__(kThreads) shift2d_tile_kernel(const __grid_constant__ ShiftArgs args) {
  using S = Smem<FT>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sR[2][2][HS_MAX_LOG2N + 1];  // [axis][start|size][level]
  __shared__ int sDoff[HS_MAX_LOG2N + 2];      // detail window offset per level (floats)
  __shared__ int sLast;

  const int g = blockIdx.y;  // face within this launch
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int n = args.log2n;
  const int m = P.m;
  if (m == 0) return;  // identity: handled by permute_kernel
  const int c = m > KF ? m - KF : 0;
  const int k = m - c;
  const int tc = (1 << c) < TC ? (1 << c) : TC;
  const int tpr = (1 << c) / tc;  // tiles per row
  if ((int)blockIdx.x >= tpr * tpr) return;
  const int i0 = (blockIdx.x / tpr) * tc;
  const int j0 = (blockIdx.x % tpr) * tc;
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in =
      args.in + (long long)b * args.in_batch_stride + (long long)f * ((long long)1 << (2 * n));
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  const int band = args.band;
  const int tid = threadIdx.x;

  float* sDet = reinterpret_cast<float*>(smem + S::DET);
  FT* sFB = reinterpret_cast<FT*>(smem + S::FB);
  FT* sFS = reinterpret_cast<FT*>(smem + S::FS);
  FT* sBig = reinterpret_cast<FT*>(smem + S::BIG);

  // ---- regions: level-m field window F_m = [2^k i0 - Q - 1, +2^k (tc+1)); P_l = parents of P_{l+1}
  if (tid < 2) {
    const int Q = tid == 0 ? P.Qy : P.Qx;
    const int o = tid == 0 ? i0 : j0;
    int s = (o << k) - Q - 1;
    int e = s + ((tc + 1) << k) - 1;
    for (int l = m - 1; l >= 0; --l) {
      s >>= 1;  // arithmetic shift = floor division for negatives
      e >>= 1;
      sR[tid][0][l] = s;
      sR[tid][1][l] = e - s + 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0;
    for (int l = 0; l < m; ++l) {
      sDoff[l] = off;
      off += 3 * (sR[0][1][l] + 1) * (sR[1][1][l] + 1);
    }
    sDoff[m] = off;
  }
  __syncthreads();

  // ---- all detail windows (parents + 1 neighbour row/column) of levels 0..m-1 in one round trip:
  //      one flat loop over every level's [3][yn+1][xn+1] window; a thread's flat index only grows,
  //      so its level pointer only moves forward; divisions by the (small) window sizes use an
  //      exact float reciprocal: floor((e + 0.5) / n) is exact for e < 2^16, n < 2^8.
  {
    const int total = sDoff[m];
    int l = -1, lend = 0, lbeg = 0, per = 1, xn = 1, ys = 0, xs = 0, mask = 0;
    float inv_per = 1.f, inv_xn = 1.f;
    for (int e = tid; e < total; e += kThreads) {
      while (e >= lend) {  // advance to the level holding e (monotone per thread)
        ++l;
        lbeg = sDoff[l];
        lend = sDoff[l + 1];
        xn = sR[1][1][l] + 1;
        per = (sR[0][1][l] + 1) * xn;
        ys = sR[0][0][l];
        xs = sR[1][0][l];
        mask = (1 << l) - 1;
        inv_per = inv_small(per);
        inv_xn = inv_small(xn);
      }
      const int loc = e - lbeg;
      const int t = div_small(loc, inv_per);
      const int rem = loc - t * per;
      const int a = div_small(rem, inv_xn);
      const int bb = rem - a * xn;
      cp_async4(sDet + e, in + (((1 + t) << (2 * l)) + (((ys + a) & mask) << l) + ((xs + bb) & mask)));
    }
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- (1) top-down l -> l+1 for l = 0 .. m-2, all three fields; level m-1 lands in sFB
  for (int l = 0; l + 1 < m; ++l) {
    const int ys = sR[0][0][l], yn = sR[0][1][l], xs = sR[1][0][l], xn = sR[1][1][l];
    const int dn = xn + 1, dplane = (yn + 1) * dn;
    const float* dt = sDet + sDoff[l];
    const FT asc = FT(pow2f(l));
    const bool dst_big = ((m - 2 - l) & 1) == 0;  // child level l+1; level m-1 -> big buffer
    FT* cf = dst_big ? sFB : sFS;
    const int cplane = dst_big ? CB * CB : CSM * CSM;
    const FT* pf = dst_big ? sFS : sFB;
    const int pplane = dst_big ? CSM * CSM : CB * CB;
    int pstride = 0, poy = 0, pox = 0;
    if (l > 0) {
      pstride = 2 * sR[1][1][l - 1];
      poy = ys - 2 * sR[0][0][l - 1];
      pox = xs - 2 * sR[1][0][l - 1];
    }
    const int cstride = 2 * xn;
    for (Walk2 w(yn * xn, xn); w.idx < yn * xn; w.next()) {
      const int pi = w.r, pj = w.c;
      FT d[2][2][2][2];  // [u][w][a][b] = delta_ab at cell (i+u, j+w)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int o = (pi + u) * dn + (pj + v);
          const FT H = FT(dt[o]) * asc, V = FT(dt[dplane + o]) * asc, D = FT(dt[2 * dplane + o]) * asc;
          d[u][v][0][0] = H + V + D;
          d[u][v][0][1] = -H + V - D;
          d[u][v][1][0] = H - V - D;
          d[u][v][1][1] = -H - V + D;
        }
      FT Xl = FT(0), Yl = FT(0), Zl = FT(0);
      if (l > 0) {
        const int po = (pi + poy) * pstride + (pj + pox);
        Xl = pf[po];
        Yl = pf[pplane + po];
        Zl = pf[2 * pplane + po];
      }
      const int co = (2 * pi) * cstride + 2 * pj;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        cf[co + a * cstride + 0] = d[0][0][a][0] - d[0][0][a][1];
        cf[co + a * cstride + 1] = Xl + d[0][0][a][1] - d[0][1][a][0];
      }
#pragma unroll
      for (int bq = 0; bq < 2; ++bq) {
        cf[cplane + co + bq] = d[0][0][0][bq] - d[0][0][1][bq];
        cf[cplane + co + cstride + bq] = Yl + d[0][0][1][bq] - d[1][0][0][bq];
      }
      cf[2 * cplane + co] = d[0][0][0][0] - d[0][0][0][1] - d[0][0][1][0] + d[0][0][1][1];  // = 4 D^
      cf[2 * cplane + co + 1] = d[0][0][0][1] - d[0][0][1][1] - d[0][1][0][0] + d[0][1][1][0];
      cf[2 * cplane + co + cstride] = d[0][0][1][0] - d[0][0][1][1] - d[1][0][0][0] + d[1][0][0][1];
      cf[2 * cplane + co + cstride + 1] = Zl + d[0][0][1][1] - d[0][1][1][0] - d[1][0][0][1] + d[1][1][0][0];
    }
    __syncthreads();
  }

  // ---- level m-1 -> m per field, fused with (2) shift and the first bottom-up step.
  //      The level-m children are stored column-parity split (sBig[c & 1][r][c >> 1]) so that the
  //      stencil's lanes read consecutive words; the shifted level-(m-1) field fld overwrites
  //      plane fld of sFB once its children are built.
  const int Sn1 = ((tc + 1) << (k - 1)) - 1;
  {
    const int l = m - 1;
    const int ys = sR[0][0][l], yn = sR[0][1][l], xs = sR[1][0][l], xn = sR[1][1][l];
    const int dn = xn + 1, dplane = (yn + 1) * dn;
    const float* dt = sDet + sDoff[l];
    const FT asc = FT(pow2f(l));
    int pstride = 0, poy = 0, pox = 0;
    if (l > 0) {
      pstride = 2 * sR[1][1][l - 1];
      poy = ys - 2 * sR[0][0][l - 1];
      pox = xs - 2 * sR[1][0][l - 1];
    }
    const int hs = xn;                   // half-row stride of the parity-split children
    const int hplane = 2 * yn * xn;      // one parity plane
    const int Cy = 2 * ys;               // unwrapped origin (rows) of the level-m window
    const int Ssy = i0 << (k - 1), Ssx = j0 << (k - 1);
    const int On = tc << (k - 1);
    const FT wy1 = FT(P.wy), wx1 = FT(P.wx);
    const FT wy0 = FT(1) - wy1, wx0 = FT(1) - wx1;
    // fused tap weights: [1,1]*[w0,w1] = [w1, 1, w0]; [1,2,1]*[w0,w1] = [w1, w0+2w1, 2w0+w1, w0]
    const FT B3y[3] = {wy1, FT(1), wy0}, B3x[3] = {wx1, FT(1), wx0};
    const FT T4y[4] = {wy1, wy0 + FT(2) * wy1, FT(2) * wy0 + wy1, wy0};
    const FT T4x[4] = {wx1, wx0 + FT(2) * wx1, FT(2) * wx0 + wx1, wx0};
    // column tap v in -1..2 lands in parity plane (v - Qx) & 1, half-column offset floor((v - Qx) / 2)
    int tapo[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) tapo[v] = ((v - 1 - P.Qx) & 1) * hplane + ((v - 1 - P.Qx) >> 1);
    const FT q = FT(0.25);
    const int lv = m - 1;
    const int gl = 1 << lv;
    const FT osc = FT(pow2f(-lv));
    const bool emit = lv < band;
    for (int fld = 0; fld < 3; ++fld) {
      const FT* pfp = sFB + fld * CB * CB;
      for (Walk2 w(yn * xn, xn); w.idx < yn * xn; w.next()) {
        const int pi = w.r, pj = w.c;
        const int o00 = pi * dn + pj;
        FT Fl = FT(0);
        if (l > 0) Fl = pfp[(pi + poy) * pstride + (pj + pox)];
        FT* ce = sBig + (2 * pi) * hs + pj;  // even child column 2pj
        FT* co = ce + hplane;                // odd child column 2pj+1
        const FT H = FT(dt[o00]) * asc, V = FT(dt[dplane + o00]) * asc, D = FT(dt[2 * dplane + o00]) * asc;
        const FT d00 = H + V + D, d01 = -H + V - D, d10 = H - V - D, d11 = -H - V + D;
        if (fld == 0) {
          const int o = o00 + 1;
          const FT Hr = FT(dt[o]) * asc, Vr = FT(dt[dplane + o]) * asc, Dr = FT(dt[2 * dplane + o]) * asc;
          const FT r00 = Hr + Vr + Dr, r10 = Hr - Vr - Dr;
          ce[0] = d00 - d01;
          co[0] = Fl + d01 - r00;
          ce[hs] = d10 - d11;
          co[hs] = Fl + d11 - r10;
        } else if (fld == 1) {
          const int o = o00 + dn;
          const FT Hb = FT(dt[o]) * asc, Vb = FT(dt[dplane + o]) * asc, Db = FT(dt[2 * dplane + o]) * asc;
          const FT b00 = Hb + Vb + Db, b01 = -Hb + Vb - Db;
          ce[0] = d00 - d10;
          co[0] = d01 - d11;
          ce[hs] = Fl + d10 - b00;
          co[hs] = Fl + d11 - b01;
        } else {
          const int o01 = o00 + 1, o10 = o00 + dn, o11 = o00 + dn + 1;
          const FT Hr = FT(dt[o01]) * asc, Vr = FT(dt[dplane + o01]) * asc, Dr = FT(dt[2 * dplane + o01]) * asc;
          const FT Hb = FT(dt[o10]) * asc, Vb = FT(dt[dplane + o10]) * asc, Db = FT(dt[2 * dplane + o10]) * asc;
          const FT Hd = FT(dt[o11]) * asc, Vd = FT(dt[dplane + o11]) * asc, Dd = FT(dt[2 * dplane + o11]) * asc;
          const FT r00 = Hr + Vr + Dr, r10 = Hr - Vr - Dr;
          const FT b00 = Hb + Vb + Db, b01 = -Hb + Vb - Db;
          const FT g00 = Hd + Vd + Dd;
          ce[0] = FT(4) * D;
          co[0] = d01 - d11 - r00 + r10;
          ce[hs] = d10 - d11 - b00 + b01;
          co[hs] = Fl + d11 - r10 - b01 + g00;
        }
      }
      __syncthreads();
      FT* dstS = sFB + fld * CB * CB;  // level m-1 field fld is dead now
      float* ob = out + (long long)gl * gl * (1 + fld);
      for (Walk2 w(Sn1 * Sn1, Sn1); w.idx < Sn1 * Sn1; w.next()) {
        const int ii = w.r, jj = w.c;
        const int gi = Ssy + ii, gj = Ssx + jj;
        const FT* base = sBig + (2 * gi - P.Qy - Cy) * hs + (gj - xs);
        FT acc = FT(0), det = FT(0);
        if (fld == 0) {  // X: rows [w1,1,w0] (u=-1..1), cols tent (v=-1..2)
#pragma unroll
          for (int u = -1; u <= 1; ++u) {
            const FT* rp = base + u * hs;
            const FT x_1 = rp[tapo[0]], x0 = rp[tapo[1]], x1 = rp[tapo[2]], x2 = rp[tapo[3]];
            acc += B3y[u + 1] * (T4x[0] * x_1 + T4x[1] * x0 + T4x[2] * x1 + T4x[3] * x2);
            det += B3y[u + 1] * (wx1 * x_1 + wx0 * x0);
          }
        } else if (fld == 1) {  // Y: rows tent (u=-1..2), cols [w1,1,w0] (v=-1..1)
#pragma unroll
          for (int u = -1; u <= 2; ++u) {
            const FT* rp = base + u * hs;
            const FT r = B3x[0] * rp[tapo[0]] + B3x[1] * rp[tapo[1]] + B3x[2] * rp[tapo[2]];
            acc += T4y[u + 1] * r;
            if (u == -1) det += wy1 * r;
            if (u == 0) det += wy0 * r;
          }
        } else {  // Z: tent x tent
#pragma unroll
          for (int u = -1; u <= 2; ++u) {
            const FT* rp = base + u * hs;
            const FT z_1 = rp[tapo[0]], z0 = rp[tapo[1]], z1 = rp[tapo[2]], z2 = rp[tapo[3]];
            acc += T4y[u + 1] * (T4x[0] * z_1 + T4x[1] * z0 + T4x[2] * z1 + T4x[3] * z2);
            const FT dr = wx1 * z_1 + wx0 * z0;
            if (u == -1) det += wy1 * dr;
            if (u == 0) det += wy0 * dr;
          }
        }
        dstS[ii * Sn1 + jj] = q * acc;
        if (ii < On && jj < On && emit)
          ob[gi * gl + gj] = (float)(q * det * osc);
      }
      __syncthreads();
    }
  }

  // ---- (3) plain bottom-up for levels m-2 .. c on the shifted windows (sFB <-> sFS)
  const FT* srcS = sFB;
  int srcN = Sn1, srcPlane = CB * CB;
  for (int lev = m - 2; lev >= c; --lev) {
    const int e = lev - c;
    const int Sn = ((tc + 1) << e) - 1;
    const int On = tc << e;
    const int Ssy = i0 << e, Ssx = j0 << e;
    const bool to_small = ((m - 2 - lev) & 1) == 0;
    FT* dst = to_small ? sFS : sFB;
    const int dstPlane = to_small ? CSM * CSM : CB * CB;
    const int gl = 1 << lev;
    const FT osc = FT(pow2f(-lev));
    const FT q = FT(0.25);
    const bool emit = lev < band;
    for (Walk2 w(Sn * Sn, Sn); w.idx < Sn * Sn; w.next()) {
      const int ii = w.r, jj = w.c;
      const int a2 = 2 * ii, b2 = 2 * jj;
      const FT* X = srcS + a2 * srcN + b2;
      const FT* Y = srcS + srcPlane + a2 * srcN + b2;
      const FT* Z = srcS + 2 * srcPlane + a2 * srcN + b2;
      const FT Xn = q * (X[0] + FT(2) * X[1] + X[2] + X[srcN] + FT(2) * X[srcN + 1] + X[srcN + 2]);
      const FT Yn = q * (Y[0] + FT(2) * Y[srcN] + Y[2 * srcN] + Y[1] + FT(2) * Y[srcN + 1] + Y[2 * srcN + 1]);
      const FT Zn = q * ((Z[0] + FT(2) * Z[1] + Z[2]) + FT(2) * (Z[srcN] + FT(2) * Z[srcN + 1] + Z[srcN + 2]) +
                         (Z[2 * srcN] + FT(2) * Z[2 * srcN + 1] + Z[2 * srcN + 2]));
      const FT hx = q * (X[0] + X[srcN]), vy = q * (Y[0] + Y[1]), dz = q * Z[0];
      dst[ii * Sn + jj] = Xn;
      dst[dstPlane + ii * Sn + jj] = Yn;
      dst[2 * dstPlane + ii * Sn + jj] = Zn;
      if (ii < On && jj < On && emit) {
        const long long o = (long long)(Ssy + ii) * gl + (Ssx + jj);
        out[(long long)gl * gl * 1 + o] = (float)(hx * osc);
        out[(long long)gl * gl * 2 + o] = (float)(vy * osc);
        out[(long long)gl * gl * 3 + o] = (float)(dz * osc);
      }
    }
    __syncthreads();
    srcS = dst;
    srcN = Sn;
    srcPlane = dstPlane;
  }
  // srcS now holds the shifted level-c fields over the owned tile (srcN = tc)

  if (blockIdx.x == 0 && tid == 0) out[0] = __ldg(in);  // scaling coefficient: unchanged (R8)
  if (c == 0) return;

  // ---- publish the owned level-c fields; the last tile of the face runs the coarse finish
  const int gc = 1 << c;
  FT* wsf = reinterpret_cast<FT*>(args.ws) + (long long)g * args.ws_face_stride;
  for (int idx = tid; idx < 3 * tc * tc; idx += kThreads) {
    const int fld = idx / (tc * tc), r = idx - fld * tc * tc;
    const int ii = r / tc, jj = r - ii * tc;
    wsf[(long long)fld * gc * gc + (long long)(i0 + ii) * gc + (j0 + jj)] = srcS[fld * srcPlane + ii * srcN + jj];
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(args.counters + g, 1u);
    sLast = (prev == (unsigned)(tpr * tpr - 1));
  }
  __syncthreads();
  if (!sLast) return;
  __threadfence();
  const long long need = 3ll * gc * gc + 3ll * (gc / 2) * (gc / 2);
  if (need * (long long)sizeof(FT) <= (long long)S::BYTES) {
    FT* A = reinterpret_cast<FT*>(smem);
    FT* B0 = A + 3 * gc * gc;
    for (int idx = tid; idx < 3 * gc * gc; idx += kThreads) A[idx] = __ldcg(wsf + idx);
    __syncthreads();
    coarse_finish<FT>(A, B0, A, c, out, band, false);
  } else {
    coarse_finish<FT>(wsf, wsf + 3ll * gc * gc, wsf, c, out, band, true);
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
      args.in + (long long)b * args.in_batch_stride + (long long)f * ((long long)1 << (2 * n));
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
hs_status launch_tiles(ShiftArgs& a, int max_tiles, cudaStream_t st) {
  static bool attr_done = false;  // idempotent attribute set (benign race: same value)
  if (!attr_done) {
    HS_CHECK_CUDA(cudaFuncSetAttribute(shift2d_tile_kernel<FT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Smem<FT>::BYTES),
                  "cudaFuncSetAttribute(shift2d_tile_kernel)");
    attr_done = true;
  }
  shift2d_tile_kernel<FT><<<dim3(max_tiles, a.num_faces), kThreads, Smem<FT>::BYTES, st>>>(a);
  HS_CHECK_LAUNCH("shift2d_tile_kernel");
  return HS_OK;
}

}  // namespace

bool shift2d_uses_fp64(int log2n) { return log2n >= 9; }

hs_status launch_shift2d(ShiftArgs& a, int max_tiles, bool any_perm, cudaStream_t st) {
  if (max_tiles > 0) {
    hs_status s = shift2d_uses_fp64(a.log2n) ? launch_tiles<double>(a, max_tiles, st)
                                             : launch_tiles<float>(a, max_tiles, st);
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
