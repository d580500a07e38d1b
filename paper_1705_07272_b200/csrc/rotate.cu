// Rotation of lat-long maps in the Haar domain: the paper's non-linear
// phase shift (algorithm).  A rotation is an elevation about X
// followed by a shift along phi; the elevation is done by the chain rule on the
// coefficients' difference fields, the shift by the exact Haar-domain shift
// (shift2d.cu).  DESIGN.md §5.9 and readings R25-R27.
//
// Map: N x N, row r at theta_r = (r + 1/2) pi / N (top first), column c at phi_c = (c + 1/2) 2 pi / N,
// p = (sin t sin f, cos t, sin t cos f); the elevation maps g(theta, phi) = f(Theta, Phi) with
// Theta = acos(R_2 p), Phi = atan2(R_1 p, R_3 p) for p' = R_x(alpha) p (eq:theta/eq:phi P:397-402).
//
//   rot_topdown_kernel   (1) the fields of f at the finest level from the detail coefficients
//                        only, level by level (X = A[i][j] - A[i][j+1], Y = A[i][j] - A[i+1][j]);
//   rot_pole_kernel      the rows of the fields across the poles (reflection: the row beyond a pole
//                        is the pole row seen from phi + pi), from the pole rows of X_f;
//   rot_chainrule_kernel (2) per output difference: X_g[i][j] = g(theta_i, phi_j) - g(theta_i, phi_j+1)
//                        and Y_g[i][j] = g(theta_i, phi_j) - g(theta_i+1, phi_j) by the chain rule
//                        (eq:pde1-2 P:416-425) with the angle increments of the two rotated
//                        samples:  dg = f_Theta dTheta + f_Phi dPhi, f_Theta = -Y_f / dtheta and
//                        f_Phi = -X_f / dphi interpolated bilinearly at the rotated midpoint
//                        (Fig. 4; R26 -- increments instead of derivatives
//                        keep the poles of the source finite);
//   (closure)            the periodic closure the Haar fields satisfy: every row of X sums to zero
//                        (Y needs none -- its last row reaches no output coefficient, only the
//                        recursion's level-0 residual; tests/test_oracle_rotate.py): the chain-rule
//                        CTAs write partial row sums, the first bottom-up level subtracts the means;
//   rot_bottomup_kernel  (3) the paper's recursion h_s = [1,1], h_t = [1,2,1], decimated by 2
//                        (eq:conv-sker P:466-478) from (X_g, Y_g, Z_g = X_g[i] - X_g[i+1])
//                        at the finest level down to level 5, one launch per level; then
//   rot_tail_kernel      levels 4 .. 0 of each map in shared memory (one launch): every detail
//                        coefficient of g;
//   rot_dc_kernel        the scaling coefficient: mean of the level-L approximation of f
//                        (L = min(n, 6), partial top-down in shared memory) resampled at the rotated
//                        positions of the N x N grid (the paper is silent), each
//                        rotated angle pair shared by a pixel and its mirror about phi = pi;
// then haar_shift's kernels move the result by beta N / (2 pi) columns.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"

namespace hs {
namespace {

constexpr int kRotChunk = 1024;   // maps per launch sequence (angles travel as kernel parameters)
constexpr int kDcLevel = 6;

struct RotParams {   // kernel parameter space holds up to 32 KB: 2 x 1024 doubles
  double ca[kRotChunk];
  double sa[kRotChunk];
};

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// ------------------------------------------------------------------------------- (1) top-down
// level l -> l+1 for all maps: fields [map][2][4^l] (X, Y) in cur, [map][2][4^(l+1)] in nxt.
__global__ void rot_topdown_kernel(const float* __restrict__ in, long long maps, int n, int l,
                                   const double* __restrict__ cur, double* __restrict__ nxt) {
  const int g = 1 << l, G2 = 2 * g;
  const long long per = 1ll << (2 * l);
  const long long total = maps * per;
  const long long NN = 1ll << (2 * n);
  const double asc = (double)pow2f(l);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e >> (2 * l);
    const int cell = (int)(e & (per - 1));
    const int i = cell >> l, j = cell & (g - 1);
    const float* src = in + b * NN;
    double d[3][4];  // cells (i,j), (i,j+1), (i+1,j): delta_00, delta_01, delta_10, delta_11
    const int cells[3] = {cell, i * g + ((j + 1) & (g - 1)), ((i + 1) & (g - 1)) * g + j};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double H = (double)__ldg(src + per + cells[k]) * asc;
      const double V = (double)__ldg(src + 2 * per + cells[k]) * asc;
      const double D = (double)__ldg(src + 3 * per + cells[k]) * asc;
      d[k][0] = H + V + D;
      d[k][1] = -H + V - D;
      d[k][2] = H - V - D;
      d[k][3] = -H - V + D;
    }
    double Xl = 0.0, Yl = 0.0;
    if (l > 0) {
      Xl = cur[b * 2 * per + cell];
      Yl = cur[b * 2 * per + per + cell];
    }
    double* X = nxt + b * 8 * per;          // [2][4 per]
    double* Y = X + 4 * per;
    const int r0 = 2 * i, c0 = 2 * j;
    // X[2i+a][2j] = d_a0 - d_a1 ;  X[2i+a][2j+1] = X_l + d_a1 - d_a0(i, j+1)
    X[r0 * G2 + c0] = d[0][0] - d[0][1];
    X[(r0 + 1) * G2 + c0] = d[0][2] - d[0][3];
    X[r0 * G2 + c0 + 1] = Xl + d[0][1] - d[1][0];
    X[(r0 + 1) * G2 + c0 + 1] = Xl + d[0][3] - d[1][2];
    // Y[2i][2j+b] = d_0b - d_1b ;  Y[2i+1][2j+b] = Y_l + d_1b - d_0b(i+1, j)
    Y[r0 * G2 + c0] = d[0][0] - d[0][2];
    Y[r0 * G2 + c0 + 1] = d[0][1] - d[0][3];
    Y[(r0 + 1) * G2 + c0] = Yl + d[0][2] - d[2][0];
    Y[(r0 + 1) * G2 + c0 + 1] = Yl + d[0][3] - d[2][1];
  }
}

// ------------------------------------------------------------------------------- (2) chain rule
// (Theta, Phi) of R_x(alpha) p(theta, phi): eq:theta / eq:phi, Phi in [0, 2 pi)
// The angle arithmetic runs in fp64: the chain rule takes differences of nearby rotated angles
// (dTheta, dPhi ~ pi / N), which fp32 resolves to only ~1e-5 relative at N = 128.
struct Ang {
  double Th, Ph;
};

// sin / cos of the half-step grid angles: theta = k pi / (2N), phi = k pi / N, k = 0 .. 2N+1
// (every sample of the chain rule -- pixel centres, neighbours, midpoints -- is on this grid)
struct Trig {
  const double* sT;
  const double* cT;
  const double* sP;
  const double* cP;
};

__global__ void rot_table_kernel(int n, double* __restrict__ tab) {
  const int N = 1 << n, K = 2 * N + 2;
  for (int k = threadIdx.x + blockIdx.x * blockDim.x; k < K; k += blockDim.x * gridDim.x) {
    double s, c;
    sincospi((double)k / (2.0 * N), &s, &c);
    tab[k] = s;
    tab[K + k] = c;
    sincospi((double)k / (double)N, &s, &c);
    tab[2 * K + k] = s;
    tab[3 * K + k] = c;
  }
}

// atan2 in fp64 to ~1e-16 absolute, without the library's special-case machinery (the chain rule
// evaluates two per rotated sample): |y| / |x| folded to t in [0, 1], t = k/8 + residual through
// atan(t) = atan(k/8) + atan(s), s = (t - c) / (1 + t c), |s| <= 1/16, and atan(s) by its Taylor
// series to s^13 (truncation s^15 / 15 < 1e-19).  One fp64 division (reciprocal + Newton).
__constant__ double kAtanK8[9] = {0.0, 0.12435499454676144, 0.24497866312686414, 0.35877067027057225,
                                  0.4636476090008061, 0.5585993153435624, 0.6435011087932844,
                                  0.7188299996216245, 0.7853981633974483};
__device__ __forceinline__ double fast_atan2(double y, double x) {
  const double ax = fabs(x), ay = fabs(y);
  const bool sw = ay > ax;
  const double mx = sw ? ay : ax, mn = sw ? ax : ay;
  if (mx == 0.0) return 0.0;
  const int k = __float2int_rn(8.f * __fdividef((float)mn, (float)mx));
  const double c = 0.125 * (double)k;
  const double num = fma(-c, mx, mn), den = fma(c, mn, mx);   // den in [mx, 2 mx]
  double r = (double)__frcp_rn((float)den);
  r = r * fma(-den, r, 2.0);
  r = r * fma(-den, r, 2.0);
  double sq = num * r;
  sq = fma(fma(-den, sq, num), r, sq);
  const double z = sq * sq;
  double pz = 1.0 / 13.0;
  pz = fma(pz, z, -1.0 / 11.0);
  pz = fma(pz, z, 1.0 / 9.0);
  pz = fma(pz, z, -1.0 / 7.0);
  pz = fma(pz, z, 1.0 / 5.0);
  pz = fma(pz, z, -1.0 / 3.0);
  double a = fma(sq * z, pz, sq) + kAtanK8[k];
  if (sw) a = 1.5707963267948966 - a;
  if (x < 0.0) a = 3.141592653589793 - a;
  return (y < 0.0) ? -a : a;
}

// rotated angles of the grid point (theta, phi) = (kt pi / 2N, kp pi / N):
// Theta = atan2(|(x', z')|, y') (= acos y' for the unit vector, better conditioned at the poles),
// Phi = atan2(x', z') in [0, 2 pi)
__device__ __forceinline__ Ang rotated_k(const Trig& tr, int kt, int kp, double ca, double sa) {
  const double st = __ldg(tr.sT + kt), ct = __ldg(tr.cT + kt), sp = __ldg(tr.sP + kp), cp = __ldg(tr.cP + kp);
  const double a = st * sp;
  const double u = ca * ct - sa * st * cp;
  const double b = sa * ct + ca * st * cp;
  Ang r;
  r.Th = fast_atan2(sqrt(fma(a, a, b * b)), u);
  double P = fast_atan2(a, b);
  if (P < 0.0) P += 6.283185307179586;
  r.Ph = P;
  return r;
}

// the same in fp32 for the DC's sample points (a mean over N^2 samples of a level-6 approximation;
// the chain rule's midpoints need fp64: an fp32 position moves a white-noise field sample by ~1e-5)
__device__ __forceinline__ void rotated_kf(const Trig& tr, int kt, int kp, float ca, float sa, float& Th, float& Ph) {
  const float st = (float)__ldg(tr.sT + kt), ct = (float)__ldg(tr.cT + kt), sp = (float)__ldg(tr.sP + kp),
              cp = (float)__ldg(tr.cP + kp);
  const float a = st * sp;
  const float u = ca * ct - sa * st * cp;
  const float b = sa * ct + ca * st * cp;
  Th = acosf(fminf(1.f, fmaxf(-1.f, u)));
  float P = atan2f(a, b);
  if (P < 0.f) P += 6.283185307179586f;
  Ph = P;
}

// bilinear sample of a field plane (rows 0..R-1) extended by the reflected rows lo (row -1) and
// hi (row R) at index coordinates (y, x), periodic in x
__device__ __forceinline__ double sample_ext(const double* __restrict__ P, const double* __restrict__ lo,
                                            const double* __restrict__ hi, int N, int R, double y, double x) {
  y = fmin(fmax(y, -1.0), (double)R);
  const double fy = floor(y), fx = floor(x);
  const double wy = y - fy, wx = x - fx;
  const int y0 = (int)fy, y1 = min(y0 + 1, R);
  const int x0 = ((int)fx) & (N - 1), x1 = (x0 + 1) & (N - 1);
  const double* r0 = y0 < 0 ? lo : (y0 >= R ? hi : P + y0 * N);
  const double* r1 = y1 < 0 ? lo : (y1 >= R ? hi : P + y1 * N);
  return (1.0 - wy) * ((1.0 - wx) * __ldg(r0 + x0) + wx * __ldg(r0 + x1)) +
         wy * ((1.0 - wx) * __ldg(r1 + x0) + wx * __ldg(r1 + x1));
}

// pole rows per map: E [map][4][N] = X row -1, X row N, Y row -1, Y row N-1 (reflected)
__global__ void rot_pole_kernel(const double* __restrict__ F, int n, double* __restrict__ E) {
  const int N = 1 << n, h = N / 2;
  const long long NN = 1ll << (2 * n);
  const double* X = F + (long long)blockIdx.x * 2 * NN;
  double* e = E + (long long)blockIdx.x * 4 * N;
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    e[c] = X[(c + h) & (N - 1)];                              // X(theta_-1, phi) = X(theta_0, phi + pi)
    e[N + c] = X[(N - 1) * N + ((c + h) & (N - 1))];
    float s0 = 0.f, s1 = 0.f;                                  // A[r][c] - A[r][c + N/2] by telescoping X
    for (int k = 0; k < h; ++k) {
      s0 += X[(c + k) & (N - 1)];
      s1 += X[(N - 1) * N + ((c + k) & (N - 1))];
    }
    e[2 * N + c] = -s0;                                        // A[-1][c] - A[0][c] = A[0][c+N/2] - A[0][c]
    e[3 * N + c] = s1;                                         // A[N-1][c] - A[N][c]
  }
}

// f's fields F [map][2][N][N] (X_f, Y_f) + pole rows E; g's fields out: G [map][2][N][N].
// One CTA per TS x TS pixel tile of one map AND its mirror tile about phi = pi: the elevation R_x
// maps phi -> 2 pi - phi to Phi -> 2 pi - Phi (Theta unchanged), so the rotated angles of every
// sample of the mirror tile are those of the left tile's samples reflected -- the CTA computes the
// rotated pixel centres (with the +1 halo rows / columns both tiles' differences need) and the two
// midpoint grids once into shared memory: 1.6 fp64 rotations per pixel instead of 3.1.  (N <= 16:
// one tile per row, its own mirror -- every sample computed.)
constexpr int kTS = 16;
__device__ __forceinline__ Ang mirror(Ang a) {
  a.Ph = (a.Ph == 0.0) ? 0.0 : 6.283185307179586 - a.Ph;
  return a;
}
__device__ __forceinline__ double chain_pixel(const double* __restrict__ Xf, const double* __restrict__ Yf,
                                              const double* __restrict__ Eb, int N, Ang A0, Ang A1x, Ang A1y, Ang Mx,
                                              Ang My, double* __restrict__ G, long long NN) {
  const double iT = (double)N * 0.3183098861837907, iP = (double)N * 0.15915494309189535;
  double xg = 0.0;
#pragma unroll
  for (int t = 0; t < 2; ++t) {   // t = 0: X_g (neighbour in phi), t = 1: Y_g (neighbour in theta)
    const Ang A1 = t ? A1y : A1x;
    const Ang M = t ? My : Mx;
    const double y = M.Th * iT - 0.5, x = M.Ph * iP - 0.5;
    const double xf = sample_ext(Xf, Eb, Eb + N, N, N, y, x - 0.5);               // X_f lives at (i, j + 1/2)
    const double yf = sample_ext(Yf, Eb + 2 * N, Eb + 3 * N, N, N - 1, y - 0.5, x);  // Y_f at (i + 1/2, j)
    const double dT = A0.Th - A1.Th;
    double dP = A0.Ph - A1.Ph;
    if (dP > 3.141592653589793) dP -= 6.283185307179586;
    if (dP < -3.141592653589793) dP += 6.283185307179586;
    const double v = -yf * dT * iT - xf * dP * iP;
    G[t * NN] = v;
    if (t == 0) xg = v;
  }
  return xg;
}

__global__ void __launch_bounds__(kTS * kTS, 4) rot_chainrule_kernel(const double* __restrict__ F, const double* __restrict__ E,
                                                                  int n, const __grid_constant__ RotParams prm, Trig tr,
                                                                  double* __restrict__ Gf, int fmaps,
                                                                  double* __restrict__ part) {
  __shared__ Ang C[kTS + 1][kTS + 2];    // centres: rows i0 .. i0 + TS, columns j0 - 1 .. j0 + TS
  __shared__ Ang MX[kTS][kTS + 1];       // X midpoints (2i + 1, 2j + 2): columns j0 - 1 .. j0 + TS - 1
  __shared__ Ang MY[kTS][kTS];           // Y midpoints (2i + 2, 2j + 1): columns j0 .. j0 + TS - 1
  const int N = 1 << n;
  const int TS = N < kTS ? N : kTS;
  const int tpr = N / TS;                          // tiles per row of the map
  const bool pair = tpr >= 2;                      // this CTA also does the mirror tile
  const int tcols = pair ? tpr / 2 : 1;
  const long long NN = 1ll << (2 * n);
  const int b = blockIdx.y;
  const int i0 = (blockIdx.x / tcols) * TS, j0 = (blockIdx.x % tcols) * TS;
  const double ca = prm.ca[b], sa = prm.sa[b];
  const int nt = TS * TS;
  const int K2 = 2 * N;                            // half-step column index modulo 2N
  // one flat index space over the three angle grids (the block's threads share the 834 rotations
  // evenly: separate loops left the first threads of each grid a rotation more than the rest)
  const int nC = (TS + 1) * (TS + 2), nX = TS * (TS + 1), nY = TS * TS;
  for (int k = threadIdx.x; k < nC + nX + nY; k += blockDim.x) {
    int kt, kp;
    Ang* dst;
    if (k < nC) {
      const int r = k / (TS + 2), c = k - r * (TS + 2) - 1;   // c = -1 .. TS
      kt = 2 * (i0 + r) + 1;
      kp = (2 * (j0 + c) + 1 + K2) % K2;
      dst = &C[r][c + 1];
    } else if (k < nC + nX) {
      const int e = k - nC, r = e / (TS + 1), c = e - r * (TS + 1) - 1;   // c = -1 .. TS - 1
      kt = 2 * (i0 + r) + 1;
      kp = (2 * (j0 + c) + 2 + K2) % K2;
      dst = &MX[r][c + 1];
    } else {
      const int e = k - nC - nX, r = e / TS, c = e - r * TS;
      kt = 2 * (i0 + r) + 2;
      kp = 2 * (j0 + c) + 1;
      dst = &MY[r][c];
    }
    *dst = rotated_k(tr, kt, kp, ca, sa);
  }
  __syncthreads();
  if (threadIdx.x >= nt) return;
  const int ti = threadIdx.x / TS, tj = threadIdx.x - ti * TS;
  const int i = i0 + ti, j = j0 + tj;
  const long long fb = fmaps ? b : 0;   // fmaps = 0: one source map shared by every rotation
  const double* Xf = F + fb * 2 * NN;
  const double* Yf = Xf + NN;
  const double* Eb = E + fb * 4 * N;
  double* G = Gf + (long long)b * 2 * NN;
  // left tile: pixel (i, j)
  double xs = chain_pixel(Xf, Yf, Eb, N, C[ti][tj + 1], C[ti][tj + 2], C[ti + 1][tj + 1], MX[ti][tj + 1],
                          MY[ti][tj], G + (long long)i * N + j, NN);
  if (pair) {   // mirror tile: pixel (i, N - 1 - j); its phi neighbour / X midpoint mirror column j - 1
    xs += chain_pixel(Xf, Yf, Eb, N, mirror(C[ti][tj + 1]), mirror(C[ti][tj]), mirror(C[ti + 1][tj + 1]),
                      mirror(MX[ti][tj]), mirror(MY[ti][tj]), G + (long long)i * N + (N - 1 - j), NN);
  }
  // the closure's row sums (R27), one partial per (map, row, tile pair) in a fixed order: the TS
  // threads of a row are an aligned group of TS lanes
  for (int o = TS >> 1; o > 0; o >>= 1) xs += __shfl_xor_sync(__activemask(), xs, o);
  if (tj == 0) part[((long long)b * N + i) * tcols + (blockIdx.x % tcols)] = xs;
}

// the closure's row mean of X_g row r (rows of X sum to zero in the Haar fields, R27)
__device__ __forceinline__ double row_mean(const double* __restrict__ part, long long b, int N, int tcols, int r) {
  const double* p = part + ((long long)b * N + r) * tcols;
  double s = 0.0;
  for (int c = 0; c < tcols; ++c) s += p[c];
  return s / (double)N;
}

// ------------------------------------------------------------------------------- (3) bottom-up
// from fields at level l+1 (src: [map][planes][4^(l+1)]; at the finest level planes = 2 and
// Z = X[i] - X[i+1]) to level l (dst [map][3][4^l]) and the level-l details of the output pyramid.
// part != nullptr (the first level, src = the chain rule's X_g, Y_g): X_g rows corrected by the
// closure's row means on load.
__global__ void rot_bottomup_kernel(const double* __restrict__ src, int src_planes, long long maps, int l,
                                    double* __restrict__ dst, float* __restrict__ out, int n,
                                    const double* __restrict__ part, int tcols) {
  const int g = 1 << l, G2 = 2 * g;
  const long long per = 1ll << (2 * l), sper = 4 * per;
  const long long total = maps * per;
  const long long NN = 1ll << (2 * n);
  const double q = 0.25, osc = (double)pow2f(-l);
  const bool zfromx = (src_planes == 2);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e >> (2 * l);
    const int cell = (int)(e & (per - 1));
    const int i = cell >> l, j = cell & (g - 1);
    const double* X = src + b * src_planes * sper;
    const double* Y = X + sper;
    const int rr[4] = {2 * i, 2 * i + 1, (2 * i + 2) & (G2 - 1), (2 * i + 3) & (G2 - 1)};
    const int cc[3] = {2 * j, 2 * j + 1, (2 * j + 2) & (G2 - 1)};
    double mr[4] = {0.0, 0.0, 0.0, 0.0};
    if (part) {
#pragma unroll
      for (int u = 0; u < 4; ++u) mr[u] = row_mean(part, b, G2, tcols, rr[u]);
    }
    auto x = [&](int u, int w) { return X[rr[u] * G2 + cc[w]] - mr[u]; };
    auto y = [&](int u, int w) { return Y[rr[u] * G2 + cc[w]]; };
    auto z = [&](int u, int w) {
      return zfromx ? x(u, w) - x(u + 1, w) : X[2 * sper + rr[u] * G2 + cc[w]];
    };
    const double Xn = q * (x(0, 0) + 2.0 * x(0, 1) + x(0, 2) + x(1, 0) + 2.0 * x(1, 1) + x(1, 2));
    const double Yn = q * (y(0, 0) + 2.0 * y(1, 0) + y(2, 0) + y(0, 1) + 2.0 * y(1, 1) + y(2, 1));
    const double Zn = q * ((z(0, 0) + 2.0 * z(0, 1) + z(0, 2)) + 2.0 * (z(1, 0) + 2.0 * z(1, 1) + z(1, 2)) +
                          (z(2, 0) + 2.0 * z(2, 1) + z(2, 2)));
    double* D = dst + b * 3 * per;
    D[cell] = Xn;
    D[per + cell] = Yn;
    D[2 * per + cell] = Zn;
    float* o = out + b * NN;
    o[per + cell] = (float)(q * (x(0, 0) + x(1, 0)) * osc);   // one rounding per output
    o[2 * per + cell] = (float)(q * (y(0, 0) + y(0, 1)) * osc);
    o[3 * per + cell] = (float)(q * z(0, 0) * osc);
  }
}


// Levels ltop-1 .. 0 of one map in shared memory (the per-level kernel's arithmetic, one launch per
// map instead of one per level): src = the level-ltop fields (2 planes + the closure's partial row
// sums when ltop = n, straight from the chain rule; else 3 planes).  ltop <= kTailTop.
constexpr int kTailTop = 5;
__global__ void __launch_bounds__(256) rot_tail_kernel(const double* __restrict__ src, int src_planes, int ltop,
                                                       float* __restrict__ out, int n, const double* __restrict__ part,
                                                       int tcols) {
  __shared__ double A[3][1 << (2 * kTailTop)];
  __shared__ double Bf[3][1 << (2 * (kTailTop - 1))];
  const long long b = blockIdx.x;
  const int G = 1 << ltop;
  const int sper = G * G;
  const long long NN = 1ll << (2 * n);
  const double* X = src + b * src_planes * (long long)sper;
  for (int e = threadIdx.x; e < sper; e += blockDim.x) {
    const int r = e >> ltop;
    A[0][e] = part ? X[e] - row_mean(part, b, G, tcols, r) : X[e];
    A[1][e] = X[sper + e];
    if (src_planes == 3) A[2][e] = X[2 * sper + e];
  }
  __syncthreads();
  if (src_planes == 2) {   // Z = X[i] - X[i + 1] of the (corrected) finest X
    for (int e = threadIdx.x; e < sper; e += blockDim.x) {
      const int r = e >> ltop, c = e & (G - 1);
      A[2][e] = A[0][e] - A[0][((r + 1) & (G - 1)) * G + c];
    }
    __syncthreads();
  }
  float* o = out + b * NN;
  for (int l = ltop - 1; l >= 0; --l) {
    const int g = 1 << l, G2 = 2 * g;
    const int per = g * g;
    const double q = 0.25, osc = (double)pow2f(-l);
    double* dX = ((ltop - 1 - l) & 1) ? &A[0][0] : &Bf[0][0];   // ping-pong: level l into Bf or A
    const int dstride = ((ltop - 1 - l) & 1) ? (1 << (2 * kTailTop)) : (1 << (2 * (kTailTop - 1)));
    const double* sX = ((ltop - 1 - l) & 1) ? &Bf[0][0] : &A[0][0];
    const int sstride = ((ltop - 1 - l) & 1) ? (1 << (2 * (kTailTop - 1))) : (1 << (2 * kTailTop));
    for (int cell = threadIdx.x; cell < per; cell += blockDim.x) {
      const int i = cell >> l, j = cell & (g - 1);
      const int rr[4] = {2 * i, 2 * i + 1, (2 * i + 2) & (G2 - 1), (2 * i + 3) & (G2 - 1)};
      const int cc[3] = {2 * j, 2 * j + 1, (2 * j + 2) & (G2 - 1)};
      auto x = [&](int u, int w) { return sX[rr[u] * G2 + cc[w]]; };
      auto y = [&](int u, int w) { return sX[sstride + rr[u] * G2 + cc[w]]; };
      auto z = [&](int u, int w) { return sX[2 * sstride + rr[u] * G2 + cc[w]]; };
      const double Xn = q * (x(0, 0) + 2.0 * x(0, 1) + x(0, 2) + x(1, 0) + 2.0 * x(1, 1) + x(1, 2));
      const double Yn = q * (y(0, 0) + 2.0 * y(1, 0) + y(2, 0) + y(0, 1) + 2.0 * y(1, 1) + y(2, 1));
      const double Zn = q * ((z(0, 0) + 2.0 * z(0, 1) + z(0, 2)) + 2.0 * (z(1, 0) + 2.0 * z(1, 1) + z(1, 2)) +
                            (z(2, 0) + 2.0 * z(2, 1) + z(2, 2)));
      dX[cell] = Xn;
      dX[dstride + cell] = Yn;
      dX[2 * dstride + cell] = Zn;
      o[per + cell] = (float)(q * (x(0, 0) + x(1, 0)) * osc);
      o[2 * per + cell] = (float)(q * (y(0, 0) + y(0, 1)) * osc);
      o[3 * per + cell] = (float)(q * z(0, 0) * osc);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------- scaling
__global__ void __launch_bounds__(256) rot_dc_kernel(const float* __restrict__ in, long long in_stride, int n,
                                                     long long map0, const __grid_constant__ RotParams prm, Trig tr,
                                                     float* __restrict__ out) {
  __shared__ float A[2][1 << (2 * kDcLevel)];
  __shared__ float red[8];
  const long long b = blockIdx.x;
  const long long NN = 1ll << (2 * n);
  const float* src = in + b * in_stride;
  const int L = n < kDcLevel ? n : kDcLevel;
  if (threadIdx.x == 0) A[0][0] = __ldg(src);
  __syncthreads();
  int cb = 0;
  for (int l = 0; l < L; ++l) {  // A_{l+1}[2i+a][2j+b] = A_l + delta_ab (averaging details = 2^l x unit)
    const int g = 1 << l, per = g * g;
    const float asc = pow2f(l);
    for (int cell = threadIdx.x; cell < per; cell += blockDim.x) {
      const int i = cell >> l, j = cell & (g - 1);
      const float H = __ldg(src + per + cell) * asc, V = __ldg(src + 2 * per + cell) * asc,
                  D = __ldg(src + 3 * per + cell) * asc;
      const float a = A[cb][cell];
      float* nx = A[cb ^ 1];
      nx[(2 * i) * 2 * g + 2 * j] = a + H + V + D;
      nx[(2 * i) * 2 * g + 2 * j + 1] = a - H + V - D;
      nx[(2 * i + 1) * 2 * g + 2 * j] = a + H - V - D;
      nx[(2 * i + 1) * 2 * g + 2 * j + 1] = a - H - V + D;
    }
    __syncthreads();
    cb ^= 1;
  }
  const int M = 1 << L;
  const int N = 1 << n;
  const double ca = prm.ca[map0 + b], sa = prm.sa[map0 + b];
  float acc = 0.f;
  const float* P = A[cb];
  auto sample = [&](float jT, float jP) {
    const float y = jT * (float)M / 3.14159265358979f - 0.5f;   // in [-1/2, M - 1/2]
    const float x = jP * (float)M / 6.283185307179586f - 0.5f;
    const float fy = floorf(y), fx = floorf(x);
    const float wy = y - fy, wx = x - fx;
    auto at = [&](int r, int c) {  // rows beyond a pole: the pole row seen from phi + pi
      if (r < 0) { r = -1 - r; c += M / 2; }
      if (r >= M) { r = 2 * M - 1 - r; c += M / 2; }
      return P[r * M + (c & (M - 1))];
    };
    const int y0 = (int)fy, x0 = (int)fx;
    return (1.f - wy) * ((1.f - wx) * at(y0, x0) + wx * at(y0, x0 + 1)) +
           wy * ((1.f - wx) * at(y0 + 1, x0) + wx * at(y0 + 1, x0 + 1));
  };
  // pixel (i, j) and its mirror (i, N - 1 - j) about phi = pi: Phi -> 2 pi - Phi (as the chain rule)
  const int hN = N / 2;
  for (long long p = threadIdx.x; p < NN / 2; p += blockDim.x) {
    const int i = (int)(p / hN), j = (int)(p - (long long)i * hN);
    float jT, jP;
    rotated_kf(tr, 2 * i + 1, 2 * j + 1, (float)ca, (float)sa, jT, jP);
    acc += sample(jT, jP);
    acc += sample(jT, jP == 0.f ? 0.f : 6.283185307179586f - jP);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    out[b * NN] = s / (float)NN;
  }
}

unsigned grid_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148ll * 32) b = 148ll * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

// tile pairs per row of the chain rule = the closure's partial row sums per row
int closure_cols(int n) { return (1 << n) >= 2 * kTS ? (1 << n) / (2 * kTS) : 1; }

// Workspace (fp64 fields: fp32 rounding of the fine differences is amplified on the coarse levels
// the recursion sums): F ping-pong 2 x [chunk][2][N^2] doubles, G [chunk][2][N^2]
// doubles, pole rows [chunk][4][N] doubles, the trig table, the pre-azimuth pyramids [maps][N^2]
// fp32, then the shift's workspace (chunk = min(maps, 1024)).
size_t rotate_workspace_bytes_impl(int log2n, long long maps) {
  const size_t NN = (size_t)1 << (2 * log2n);
  const size_t mc = (size_t)(maps < kRotChunk ? maps : kRotChunk);
  const size_t fd = (mc * 2 * NN * sizeof(double) + 255) & ~size_t(255);
  const size_t pb = (mc * 4 * ((size_t)1 << log2n) * sizeof(double) + 255) & ~size_t(255);
  const size_t tb = (4 * (2 * ((size_t)1 << log2n) + 2) * sizeof(double) + 255) & ~size_t(255);
  const size_t tp = ((size_t)maps * NN * sizeof(float) + 255) & ~size_t(255);
  const size_t pr = (mc * ((size_t)1 << log2n) * (size_t)closure_cols(log2n) * sizeof(double) + 255) & ~size_t(255);
  return 3 * fd + pb + tb + tp + pr + ((shift_workspace_bytes_impl(2, log2n, maps) + 255) & ~size_t(255));
}

hs_status launch_rotate(const float* in, float* out, int n, long long maps, const double* angles, void* ws,
                        size_t ws_bytes, cudaStream_t st, bool bcast) {
  const long long NN = 1ll << (2 * n);
  const size_t mcap = (size_t)(maps < kRotChunk ? maps : kRotChunk);
  const size_t fd = (mcap * 2 * (size_t)NN * sizeof(double) + 255) & ~size_t(255);
  const size_t pb = (mcap * 4 * ((size_t)1 << n) * sizeof(double) + 255) & ~size_t(255);
  const int K = 2 * (1 << n) + 2;
  const size_t tb = (4 * (size_t)K * sizeof(double) + 255) & ~size_t(255);
  const size_t tp = ((size_t)maps * NN * sizeof(float) + 255) & ~size_t(255);
  char* base = reinterpret_cast<char*>(ws);
  double* bufA = reinterpret_cast<double*>(base);
  double* bufB = reinterpret_cast<double*>(base + fd);
  double* Gf = reinterpret_cast<double*>(base + 2 * fd);
  double* poles = reinterpret_cast<double*>(base + 3 * fd);
  double* tab = reinterpret_cast<double*>(base + 3 * fd + pb);
  float* tmp = reinterpret_cast<float*>(base + 3 * fd + pb + tb);
  const int tcols = closure_cols(n);
  const size_t pr = (mcap * ((size_t)1 << n) * (size_t)tcols * sizeof(double) + 255) & ~size_t(255);
  double* part = reinterpret_cast<double*>(base + 3 * fd + pb + tb + tp);
  void* sws = base + 3 * fd + pb + tb + tp + pr;
  const size_t sws_bytes = ws_bytes - (3 * fd + pb + tb + tp + pr);
  rot_table_kernel<<<(K + 255) / 256, 256, 0, st>>>(n, tab);
  HS_CHECK_LAUNCH("rot_table_kernel");
  const Trig tr{tab, tab + K, tab + 2 * K, tab + 3 * K};

  for (long long m0 = 0; m0 < maps; m0 += kRotChunk) {
    const long long mc = (maps - m0) < kRotChunk ? (maps - m0) : kRotChunk;
    RotParams prm;
    for (long long k = 0; k < mc; ++k) {
      prm.ca[k] = std::cos(angles[2 * (m0 + k)]);
      prm.sa[k] = std::sin(angles[2 * (m0 + k)]);
    }
    // bcast: every map rotates the same source pyramid -- its fields and pole rows are built once
    const float* src = bcast ? in : in + m0 * NN;
    const long long mf = bcast ? 1 : mc;
    float* dtmp = tmp + m0 * NN;
    // (1) top-down to the finest fields (ping-pong between bufA and bufB)
    double* cur = bufB;
    for (int l = 0; l < n; ++l) {
      double* nxt = (cur == bufA) ? bufB : bufA;
      rot_topdown_kernel<<<grid_for(mf << (2 * l)), 256, 0, st>>>(src, mf, n, l, cur, nxt);
      HS_CHECK_LAUNCH("rot_topdown_kernel");
      cur = nxt;
    }
    // (2) pole rows, chain rule, closure
    rot_pole_kernel<<<(unsigned)mf, 256, 0, st>>>(cur, n, poles);
    HS_CHECK_LAUNCH("rot_pole_kernel");
    {
      const int TS = (1 << n) < kTS ? (1 << n) : kTS;
      const int tpr = (1 << n) / TS;
      const int ctas = (tpr >= 2 ? tpr / 2 : 1) * tpr;   // tile pairs (mirror about phi = pi)
      rot_chainrule_kernel<<<dim3(ctas, (unsigned)mc), kTS * kTS, 0, st>>>(cur, poles, n, prm, tr, Gf, bcast ? 0 : 1,
                                                                           part);
    }
    HS_CHECK_LAUNCH("rot_chainrule_kernel");
    // (3) bottom-up, every detail level of the rotated pyramid; the closure (R27) is applied as
    // the first level loads X_g (row means from the chain rule's partial sums); levels below
    // kTailTop in one launch per chunk
    if (n <= kTailTop) {
      rot_tail_kernel<<<(unsigned)mc, 256, 0, st>>>(Gf, 2, n, dtmp, n, part, tcols);
      HS_CHECK_LAUNCH("rot_tail_kernel");
    } else {
      const double* s = Gf;
      int planes = 2;
      double* d = bufA;
      const double* pp = part;
      for (int l = n - 1; l >= kTailTop; --l) {
        rot_bottomup_kernel<<<grid_for(mc << (2 * l)), 256, 0, st>>>(s, planes, mc, l, d, dtmp, n, pp, tcols);
        HS_CHECK_LAUNCH("rot_bottomup_kernel");
        pp = nullptr;
        s = d;
        planes = 3;
        d = (d == bufA) ? bufB : bufA;
      }
      rot_tail_kernel<<<(unsigned)mc, 256, 0, st>>>(s, 3, kTailTop, dtmp, n, nullptr, 0);
      HS_CHECK_LAUNCH("rot_tail_kernel");
    }
    rot_dc_kernel<<<(unsigned)mc, 256, 0, st>>>(src, bcast ? 0 : NN, n, 0, prm, tr, dtmp);
    HS_CHECK_LAUNCH("rot_dc_kernel");
  }
  // azimuth: the exact shift by beta N / (2 pi) columns
  std::vector<double> sh((size_t)maps * 2);
  for (long long k = 0; k < maps; ++k) {
    sh[2 * k] = 0.0;
    sh[2 * k + 1] = angles[2 * k + 1] * (double)(1 << n) / 6.283185307179586;
  }
  return launch_shift(tmp, out, 2, n, 1, maps, NN, NN, sh.data(), nullptr, nullptr, n, sws, sws_bytes, st);
}

}  // namespace hs
