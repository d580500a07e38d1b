// Fused per-vertex shift + relight at N = 128 by residue planes (DESIGN.md
// §5.5).  r_v = < S_{s_v} L , T_v >.
//
// The shift of a difference field F at the finest level is the box projection
//   S F = sum_{a,b in {0,1}} w^y_a w^x_b roll(F, (q_y + a, q_x + b)),   w_0 = 1 - phi, w_1 = phi,
// and the bottom-up BU (the paper's [1,1] x [1,2,1] recursion) is linear and
// commutes with rolls by even amounts:  BU(roll(X, 2R)) = roll(BU(X), R).  Hence for Q = q + (a, b)
//   BU^k(roll(F, Q)) = roll(P_{k, Q mod 2^k}, Q div 2^k),   P_{k, rho} = BU(roll(P_{k-1, rho mod 2^(k-1)},
//                                                                     rho div 2^(k-1)))
// -- a light-only precomputation over the 4^k residues rho.  Per vertex, the level n-1 and n-2
// outputs are then four rolled reads of precomputed planes instead of a shift + stencil:
//   planes_kernel   (per face and field, fp64): D1[4][64][64] (level n-1 details), D2[16][32][32]
//                   (level n-2 details), F2[16][32][32] (level n-2 fields), scales folded in;
//   planes3_kernel  D3[64][16][16] and F3 (level n-3 details and fields) from F2;
//   planes_low_kernel DL: the details of levels n-4 .. 0, 4^n values per level (residues x cells);
//   planes_a_kernel one warp per vertex: sum_ab w_ab (< T_{n-1}, roll(D1_ab) > + < T_{n-2}, roll(D2_ab) >)
//                   (D1 rows doubled in shared memory so a warp's 64 rows never wrap; HBM-bound);
//   planes_c_kernel one warp per vertex: levels n-3 .. 0 the same way (D3 in shared memory, DL gathered
//                   from L2 one vertex ahead with the T values) -- no per-vertex bottom-up;
//   finish          r_v = the 2 x 3F partials + sum_f T_v[f][0] L_f[0].
// No block barriers after the plane fills: every warp owns its vertex.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {

constexpr int kPN = 7;                    // log2 N of this path
constexpr int kPG = 64;                   // level n-1 side
constexpr int kPD1 = 4 * kPG * kPG;       // D1 floats
constexpr int kPD2 = 16 * 32 * 32;        // D2 (and F2) floats
constexpr int kPD3 = 2 * 64 * 16 * 16;    // level n-3 details D3[64][256], then fields F3[64][256]
constexpr int kPL = 1 << (2 * kPN);       // one residue-plane level below n-3: 4^k residues x 4^(n-k) cells
constexpr int kPDL = 4 * kPL;             // details of levels n-4 .. 0 (k = 4 .. 7)
constexpr int kPlanesPerUnit = kPD1 + 2 * kPD2 + kPD3 + kPDL;

namespace {

__device__ __forceinline__ float pw2(int e) { return __int_as_float((127 + e) << 23); }

// one bottom-up cell (level LEV from the periodic plane src of side 2^(LEV+1) rolled by (ry, rx)):
// the shifted field fv and the detail dv before its 2^-LEV scale (FLD: 0 = X -> H, 1 = Y -> V, 2 = Z -> D)
template <typename V, int FLD>
__device__ __forceinline__ void bu_rolled(const V* src, int Gs, int i, int j, int ry, int rx, V& fv, V& dv) {
  const int m = Gs - 1;
  const V* p0 = src + ((2 * i - ry) & m) * Gs;
  const V* p1 = src + ((2 * i + 1 - ry) & m) * Gs;
  const V* p2 = src + ((2 * i + 2 - ry) & m) * Gs;
  const int c0 = (2 * j - rx) & m, c1 = (2 * j + 1 - rx) & m, c2 = (2 * j + 2 - rx) & m;
  const V q = V(0.25);
  if (FLD == 0) {
    fv = q * (p0[c0] + V(2) * p0[c1] + p0[c2] + p1[c0] + V(2) * p1[c1] + p1[c2]);
    dv = q * (p0[c0] + p1[c0]);
  } else if (FLD == 1) {
    fv = q * (p0[c0] + V(2) * p1[c0] + p2[c0] + p0[c1] + V(2) * p1[c1] + p2[c1]);
    dv = q * (p0[c0] + p0[c1]);
  } else {
    fv = q * ((p0[c0] + V(2) * p0[c1] + p0[c2]) + V(2) * (p1[c0] + V(2) * p1[c1] + p1[c2]) +
              (p2[c0] + V(2) * p2[c1] + p2[c2]));
    dv = q * p0[c0];
  }
}

// ------------------------------------------------------------------------------- precompute
// fields64: the fp64 level-n fields [f][3][N][N] (natural layout) at stride face_stride doubles
template <int FLD>
__device__ void planes_body(const double* F, float* out, double* F1) {
  // level n-1, residues rho in {0,1}^2:  P_{1,rho} = BU(roll(F, rho))
  for (int idx = threadIdx.x; idx < 4 * kPG * kPG; idx += blockDim.x) {
    const int rho = idx >> 12, cell = idx & 4095, i = cell >> 6, j = cell & 63;
    double fv, dv;
    bu_rolled<double, FLD>(F, 128, i, j, rho >> 1, rho & 1, fv, dv);
    F1[idx] = fv;
    out[idx] = (float)(dv * (double)pw2(-(kPN - 1)));
  }
  __syncthreads();
  // level n-2, residues rho' in {0..3}^2:  P_{2,rho'} = BU(roll(P_{1, rho' mod 2}, rho' div 2))
  float* D2 = out + kPD1;
  float* F2 = D2 + kPD2;
  for (int idx = threadIdx.x; idx < kPD2; idx += blockDim.x) {
    const int rho = idx >> 10, cell = idx & 1023, i = cell >> 5, j = cell & 31;
    const int ry = rho >> 2, rx = rho & 3;
    double fv, dv;
    bu_rolled<double, FLD>(F1 + (((ry & 1) << 1) | (rx & 1)) * 4096, 64, i, j, ry >> 1, rx >> 1, fv, dv);
    D2[idx] = (float)(dv * (double)pw2(-(kPN - 2)));
    F2[idx] = (float)fv;
  }
}

__global__ void __launch_bounds__(512) planes_kernel(const double* __restrict__ fields64, long long face_stride,
                                                     float* __restrict__ planes) {
  extern __shared__ double F1s[];   // [4][64][64] fp64 level n-1 fields of the four residues
  const int f = blockIdx.x / 3, t = blockIdx.x % 3;
  const double* F = fields64 + (long long)f * face_stride + (long long)t * (1 << (2 * kPN));
  float* out = planes + (long long)blockIdx.x * kPlanesPerUnit;
  if (t == 0) planes_body<0>(F, out, F1s);
  else if (t == 1) planes_body<1>(F, out, F1s);
  else planes_body<2>(F, out, F1s);
}

// level n-3, residues rho'' in {0..7}^2:  P_{3,rho''} = BU(roll(P_{2, rho'' mod 4}, rho'' div 4)), from
// the (fp32) level n-2 fields F2 of planes_kernel
template <int FLD>
__device__ void planes3_body(const float* F2, float* D3, float* F3) {
  for (int idx = threadIdx.x; idx < 64 * 256; idx += blockDim.x) {
    const int rho = idx >> 8, cell = idx & 255, i = cell >> 4, j = cell & 15;
    const int ry = rho >> 3, rx = rho & 7;
    float fv, dv;
    bu_rolled<float, FLD>(F2 + (((ry & 3) << 2) | (rx & 3)) * 1024, 32, i, j, ry >> 2, rx >> 2, fv, dv);
    D3[idx] = dv * pw2(-(kPN - 3));
    F3[idx] = fv;
  }
}

__global__ void __launch_bounds__(256) planes3_kernel(float* __restrict__ planes) {
  const int t = blockIdx.x % 3;
  float* base = planes + (long long)blockIdx.x * kPlanesPerUnit;
  const float* F2 = base + kPD1 + kPD2;
  float* D3 = base + kPD1 + 2 * kPD2;
  if (t == 0) planes3_body<0>(F2, D3, D3 + kPD3 / 2);
  else if (t == 1) planes3_body<1>(F2, D3, D3 + kPD3 / 2);
  else planes3_body<2>(F2, D3, D3 + kPD3 / 2);
}

// levels n-4 .. 0 (k = 4 .. 7): P_{k,rho} = BU(roll(P_{k-1, rho mod 2^(k-1)}, rho div 2^(k-1))) over
// the 4^k residues rho, each a 2^(n-k) square: 4^n values per level, ping-ponged in shared memory
// (fields) from F3; the details (scaled to unit-square) go to DL[k - 4].
template <int FLD>
__device__ void planes_low_body(const float* __restrict__ F3, float* __restrict__ DL, float* Fa, float* Fb) {
  for (int idx = threadIdx.x; idx < kPL; idx += blockDim.x) Fa[idx] = F3[idx];
  __syncthreads();
  const float* src = Fa;
  float* dst = Fb;
#pragma unroll 1
  for (int k = 4; k <= kPN; ++k) {
    const int l = kPN - k, side = 1 << l, rk = 1 << k, rh = rk >> 1;   // cells side^2, residues rk^2
    for (int idx = threadIdx.x; idx < kPL; idx += blockDim.x) {
      const int rho = idx >> (2 * l), cell = idx & (side * side - 1);
      const int ry = rho >> k, rx = rho & (rk - 1);
      const int i = cell >> l, j = cell & (side - 1);
      const int parent = ((ry & (rh - 1)) << (k - 1)) | (rx & (rh - 1));
      float fv, dv;
      bu_rolled<float, FLD>(src + parent * (4 * side * side), 2 * side, i, j, ry >> (k - 1), rx >> (k - 1), fv, dv);
      DL[(k - 4) * kPL + idx] = dv * pw2(-l);
      dst[idx] = fv;
    }
    __syncthreads();
    const float* t = src;
    src = dst;
    dst = const_cast<float*>(t);
  }
}

__global__ void __launch_bounds__(512) planes_low_kernel(float* __restrict__ planes) {
  extern __shared__ float smL[];   // two field ping-pong buffers of kPL floats
  const int t = blockIdx.x % 3;
  float* base = planes + (long long)blockIdx.x * kPlanesPerUnit;
  const float* F3 = base + kPD1 + 2 * kPD2 + kPD3 / 2;
  float* DL = base + kPD1 + 2 * kPD2 + kPD3;
  if (t == 0) planes_low_body<0>(F3, DL, smL, smL + kPL);
  else if (t == 1) planes_low_body<1>(F3, DL, smL, smL + kPL);
  else planes_low_body<2>(F3, DL, smL, smL + kPL);
}

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds(uint32_t a) {
  float x;
  asm("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));   // planes are read-only after the fill
  return x;
}

// ------------------------------------------------------------------------------- level n-1
constexpr int kAWarps = 32;
constexpr int kARows = 2 * kPG;   // D1 rows doubled: rows s .. s+63 never wrap
constexpr int kASmem = (4 * kARows * kPG + kPD2) * 4;   // D1 doubled + D2

__global__ void __launch_bounds__(kAWarps * 32, 1)
    planes_a_kernel(const float* __restrict__ T, long long V, int faces, const float* __restrict__ planes,
                    const int4* __restrict__ vparams, float* __restrict__ partial, int nsplit) {
  extern __shared__ __align__(16) float D1s[];   // [4][128][64]
  const int units = 3 * faces;
  const int unit = blockIdx.x % units, split = blockIdx.x / units;
  const int f = unit / 3, t = unit - 3 * (unit / 3);
  const float* src = planes + (long long)unit * kPlanesPerUnit;
  for (int idx = threadIdx.x; idx < 4 * kARows * kPG; idx += blockDim.x) {
    const int rho = idx / (kARows * kPG), rem = idx - rho * (kARows * kPG);
    const int r = rem >> 6, c = rem & 63;
    D1s[idx] = __ldg(src + rho * 4096 + (r & 63) * 64 + c);
  }
  float* D2s = D1s + 4 * kARows * kPG;
  for (int idx = threadIdx.x; idx < kPD2; idx += blockDim.x) D2s[idx] = __ldg(src + kPD1 + idx);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long NN = 1ll << (2 * kPN);
  const long long Kt = (long long)faces * NN;
  const long long v0 = V * split / nsplit, v1 = V * (split + 1) / nsplit;
  const uint32_t base = saddr(D1s);
  for (long long v = v0 + warp; v < v1; v += kAWarps) {
    const int4 pr = __ldg(vparams + v);
    const float wy1 = __int_as_float(pr.z), wx1 = __int_as_float(pr.w);
    const float* Tl = T + v * Kt + (long long)f * NN + (long long)(1 + t) * 4096 + lane;
    // combo (a, b): Q = q + (a, b) mod N; residue Q & 1, roll Q >> 1
    uint32_t ad[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int Qy = (pr.x + a) & 127;
      const int s = (-(Qy >> 1)) & 63;   // D1 row of output row 0
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int Qx = (pr.y + b) & 127;
        const int rho = ((Qy & 1) << 1) | (Qx & 1);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          ad[a][b][c] = base + (uint32_t)(((rho * kARows + s) * 64 + ((lane + 32 * c - (Qx >> 1)) & 63)) * 4);
      }
    }
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll 8
    for (int i = 0; i < kPG; ++i) {
      const float t0 = __ldg(Tl + i * 64), t1 = __ldg(Tl + i * 64 + 32);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          acc[a][b] = fmaf(t0, lds(ad[a][b][0] + i * 256), acc[a][b]);
          acc[a][b] = fmaf(t1, lds(ad[a][b][1] + i * 256), acc[a][b]);
        }
    }
    // level n-2 details: residue Q & 3, roll Q >> 2; lanes = columns (conflict-free), rows wrapped
    const float* T2 = T + v * Kt + (long long)f * NN + (long long)(1 + t) * 1024 + lane;
    int off2[2][2], ry2[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      ry2[a] = ((pr.x + a) & 127) >> 2;
#pragma unroll
      for (int b = 0; b < 2; ++b)
        off2[a][b] = ((((pr.x + a) & 3) << 2) | ((pr.y + b) & 3)) * 1024 + ((lane - (((pr.y + b) & 127) >> 2)) & 31);
    }
    float acc2[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const float t2 = __ldg(T2 + i * 32);
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int row = ((i - ry2[a]) & 31) * 32;
#pragma unroll
        for (int b = 0; b < 2; ++b) acc2[a][b] = fmaf(t2, D2s[off2[a][b] + row], acc2[a][b]);
      }
    }
    const float wy0 = 1.f - wy1, wx0 = 1.f - wx1;
    float r = wy0 * (wx0 * (acc[0][0] + acc2[0][0]) + wx1 * (acc[0][1] + acc2[0][1])) +
              wy1 * (wx0 * (acc[1][0] + acc2[1][0]) + wx1 * (acc[1][1] + acc2[1][1]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0) partial[v * 2 * units + unit] = r;
  }
}

// ------------------------------------------------------------------------------- level n-3 .. 0
// Levels n-3 .. 0 of one unit per vertex: four rolled reads of the residue planes per output cell
// (level n-3 from shared memory, levels n-4 .. 0 from the L2-resident DL), no bottom-up.  The T
// values and the DL gathers of the next vertex are in flight while the current one is reduced.
constexpr int kCWarps = 16;
constexpr int kCSmem = kPD3 * 4;   // D3[64][32][16]: rows doubled so a lane's 8 rows never wrap

struct CTvals {
  float t3[8];      // level n-3 T: cells lane + 32 k
  float t4[2];      // level n-4 T: cells lane, lane + 32
  float tl[3];      // levels 2, 1, 0 (n = 7) T: cell lane & 15 / lane & 3 / 0, zero on duplicate lanes
  float g4[2][4];   // level n-4 plane values per cell and combo (a, b)
  float gl[3][4];   // levels 2, 1, 0 plane values per combo
  int4 pr;
};
// plane value of level L (k = kPN - L) cell (i, j) for combo Q = (qy, qx): residue (Q mod 2^k), roll
// Q div 2^k (the residue / roll part is the same for every lane of the warp)
template <int L>
__device__ __forceinline__ float low_gather(const float* __restrict__ DL, int qy, int qx, int i, int j) {
  constexpr int k = kPN - L, side = 1 << L;
  const int rho = ((qy & ((1 << k) - 1)) << k) | (qx & ((1 << k) - 1));
  return __ldg(DL + (k - 4) * kPL + rho * side * side + (((i - (qy >> k)) & (side - 1)) << L) +
               ((j - (qx >> k)) & (side - 1)));
}
__device__ __forceinline__ void planes_c_load(CTvals& c, const float* __restrict__ Tv, int fld,
                                              const int4* __restrict__ vp, const float* __restrict__ DL, int lane) {
  c.pr = __ldg(vp);
#pragma unroll
  for (int k = 0; k < 8; ++k) c.t3[k] = __ldg(Tv + (1 + fld) * 256 + lane + 32 * k);
  c.t4[0] = __ldg(Tv + (1 + fld) * 64 + lane);
  c.t4[1] = __ldg(Tv + (1 + fld) * 64 + 32 + lane);
  const int c2 = lane & 15, c1 = lane & 3;
  c.tl[0] = __ldg(Tv + (1 + fld) * 16 + c2);
  c.tl[1] = __ldg(Tv + (1 + fld) * 4 + c1);
  c.tl[2] = __ldg(Tv + (1 + fld));
  if (lane >= 16) c.tl[0] = 0.f;   // each cell counted by one lane
  if (lane >= 4) c.tl[1] = 0.f;
  if (lane >= 1) c.tl[2] = 0.f;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int qy = (c.pr.x + a) & 127, qx = (c.pr.y + b) & 127;
      c.g4[0][2 * a + b] = low_gather<3>(DL, qy, qx, lane >> 3, lane & 7);
      c.g4[1][2 * a + b] = low_gather<3>(DL, qy, qx, (lane >> 3) + 4, lane & 7);
      c.gl[0][2 * a + b] = low_gather<2>(DL, qy, qx, c2 >> 2, c2 & 3);
      c.gl[1][2 * a + b] = low_gather<1>(DL, qy, qx, c1 >> 1, c1 & 1);
      c.gl[2][2 * a + b] = low_gather<0>(DL, qy, qx, 0, 0);
    }
}

__device__ __forceinline__ float planes_c_vertex(uint32_t d3base, const CTvals& cv, int lane) {
  const int4 pr = cv.pr;
  const float wy1 = __int_as_float(pr.z), wx1 = __int_as_float(pr.w), wy0 = 1.f - wy1, wx0 = 1.f - wx1;
  const float w[4] = {wy0 * wx0, wy0 * wx1, wy1 * wx0, wy1 * wx1};
  // level n-3: cell lane + 32 k = (row 2k + lane / 16, column lane % 16), combo residue Q & 7, roll
  // Q >> 3: a half-warp reads one rolled 16-wide row; with the doubled rows, row 2k + rs_a of the
  // residue plane is an immediate offset (128 k bytes) from the combo's base
  const int jl = lane & 15, il = lane >> 4;
  uint32_t ad[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int qy = (pr.x + a) & 127;
    const int rs = (il - (qy >> 3)) & 15;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int qx = (pr.y + b) & 127;
      const int rho = ((qy & 7) << 3) | (qx & 7);
      ad[a][b] = d3base + (uint32_t)(((rho * 32 + rs) * 16 + ((jl - (qx >> 3)) & 15)) * 4);
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float d = 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) d = fmaf(w[2 * a + b], lds(ad[a][b] + 128 * k), d);
    acc = fmaf(d, cv.t3[k], acc);
  }
  // levels n-4 .. 0 from the gathered plane values
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float d = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) d = fmaf(w[c], cv.g4[h][c], d);
    acc = fmaf(d, cv.t4[h], acc);
  }
#pragma unroll
  for (int h = 0; h < 3; ++h) {
    float d = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) d = fmaf(w[c], cv.gl[h][c], d);
    acc = fmaf(d, cv.tl[h], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__global__ void __launch_bounds__(kCWarps * 32, 1)
    planes_c_kernel(const float* __restrict__ T, long long V, int faces, const float* __restrict__ planes,
                    const int4* __restrict__ vparams, float* __restrict__ partial, int nsplit) {
  extern __shared__ __align__(16) float D3s[];
  const int units = 3 * faces;
  const int unit = blockIdx.x % units, split = blockIdx.x / units;
  const int f = unit / 3, t = unit - 3 * (unit / 3);
  const float* src = planes + (long long)unit * kPlanesPerUnit + kPD1 + 2 * kPD2;
  const float* DL = src + kPD3;
  for (int idx = threadIdx.x; idx < kPD3; idx += blockDim.x) {   // [rho][row 0..31][col] <- [rho][row & 15][col]
    const int rho = idx >> 9, r = (idx >> 4) & 31, c = idx & 15;
    D3s[idx] = __ldg(src + rho * 256 + (r & 15) * 16 + c);
  }
  __syncthreads();
  const uint32_t d3base = saddr(D3s);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long NN = 1ll << (2 * kPN);
  const long long Kt = (long long)faces * NN;
  const long long v0 = V * split / nsplit, v1 = V * (split + 1) / nsplit;
  // software pipeline: the next vertex's T values, parameters and plane gathers are in flight
  CTvals cur, nxt;
  if (v0 + warp < v1) planes_c_load(nxt, T + (v0 + warp) * Kt + (long long)f * NN, t, vparams + v0 + warp, DL, lane);
  for (long long v = v0 + warp; v < v1; v += kCWarps) {
    cur = nxt;
    if (v + kCWarps < v1)
      planes_c_load(nxt, T + (v + kCWarps) * Kt + (long long)f * NN, t, vparams + v + kCWarps, DL, lane);
    const float r = planes_c_vertex(d3base, cur, lane);
    if (lane == 0) partial[v * 2 * units + units + unit] = r;
  }
}

__global__ void planes_finish_kernel(const float* __restrict__ partial, const float* __restrict__ T,
                                     const float* __restrict__ light, long long V, int faces, float* __restrict__ R) {
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int units = 3 * faces;
  const long long NN = 1ll << (2 * kPN);
  float s = 0.f;
  for (int u = 0; u < 2 * units; ++u) s += partial[v * 2 * units + u];
  for (int f = 0; f < faces; ++f) s = fmaf(__ldg(T + v * faces * NN + f * NN), __ldg(light + f * NN), s);
  R[v] = s;
}

int sm_count() { return device_sm_count(); }

// ------------------------------------------------------------------------------- N <= 64: every level
// For small faces every level's residue planes fit in shared memory at once (n levels x 4^n
// values: 96 KB at N = 64), so the per-vertex work is only rolled plane reads:
//   r_v(unit) = sum_l sum_ab w_ab < T_l, roll(D_{l, Q_ab mod 2^(n-l)}, Q_ab div 2^(n-l)) >
// with no shift, no stencil and no bottom-up per vertex.  D_l layout per unit and level:
// [rho_y][rho_x][2^l][2^l] (4^n floats), levels n-1 .. 0 concatenated.

// residue planes of every level of one (face, field), fp64 recursion in shared memory
template <int FLD>
__device__ void small_planes_body(const double* F, int n, float* out, double* A, double* Bf) {
  const int NN = 1 << (2 * n);
  const double* src = F;   // level n fields (one residue)
  double* dst = A;
  for (int k = 1; k <= n; ++k) {
    const int l = n - k, g = 1 << l, gg = g * g, R = 1 << k;       // output level, side, residues per axis
    const int Gs = 2 * g, Rp = R >> 1;                             // source side, source residues per axis
    float* D = out + (long long)(k - 1) * NN;
    for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) {
      const int rho = idx / gg, cell = idx - rho * gg;
      const int ry = rho / R, rx = rho - ry * R;
      const int i = cell >> l, j = cell & (g - 1);
      const double* S = src + (long long)((ry % Rp) * Rp + (rx % Rp)) * (Gs * Gs);
      double fv, dv;
      bu_rolled<double, FLD>(S, Gs, i, j, ry / Rp, rx / Rp, fv, dv);
      dst[idx] = fv;
      D[idx] = (float)(dv * (double)pw2(-l));
    }
    __syncthreads();
    src = dst;
    dst = (dst == A) ? Bf : A;
  }
}

__global__ void __launch_bounds__(512) small_planes_kernel(const double* __restrict__ fields64, long long face_stride,
                                                           int n, float* __restrict__ planes) {
  extern __shared__ double sp[];   // two 4^n ping-pong planes (fp64)
  const int f = blockIdx.x / 3, t = blockIdx.x % 3;
  const int NN = 1 << (2 * n);
  const double* F = fields64 + (long long)f * face_stride + (long long)t * NN;
  float* out = planes + (long long)blockIdx.x * n * NN;
  if (t == 0) small_planes_body<0>(F, n, out, sp, sp + NN);
  else if (t == 1) small_planes_body<1>(F, n, out, sp, sp + NN);
  else small_planes_body<2>(F, n, out, sp, sp + NN);
}

constexpr int kSWarps = 32;

template <int LOG2N>
__global__ void __launch_bounds__(kSWarps * 32)
    small_relight_kernel(const float* __restrict__ T, long long V, int faces, const float* __restrict__ planes,
                         const int4* __restrict__ vparams, float* __restrict__ partial, int nsplit) {
  constexpr int n = LOG2N, NN = 1 << (2 * n);
  extern __shared__ __align__(16) float Ds[];   // [n][4^n]: levels n-1 .. 0
  const int units = 3 * faces;
  const int unit = blockIdx.x % units, split = blockIdx.x / units;
  const int f = unit / 3, t = unit - 3 * (unit / 3);
  const float* src = planes + (long long)unit * n * NN;
  for (int idx = threadIdx.x; idx < n * NN; idx += blockDim.x) Ds[idx] = __ldg(src + idx);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long Kt = (long long)faces * NN;
  const long long v0 = V * split / nsplit, v1 = V * (split + 1) / nsplit;
  for (long long v = v0 + warp; v < v1; v += kSWarps) {
    const int4 pr = __ldg(vparams + v);
    const float* Tv = T + v * Kt + (long long)f * NN;
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
    for (int k = 1; k <= n; ++k) {
      const int l = n - k, g = 1 << l, gg = g * g, R = 1 << k;
      const float* D = Ds + (k - 1) * NN;
      const float* Tl = Tv + (long long)(1 + t) * gg;
      int ry[2], rx[2], py[2], px[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int Qy = (pr.x + a) & ((1 << n) - 1), Qx = (pr.y + a) & ((1 << n) - 1);
        py[a] = Qy & (R - 1);
        ry[a] = Qy >> k;
        px[a] = Qx & (R - 1);
        rx[a] = Qx >> k;
      }
      const float* Db[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) Db[a][b] = D + (py[a] * R + px[b]) * gg;
#pragma unroll 8   // T loads of several cells in flight (the HBM latency, not the arithmetic, bounds this)
      for (int idx = lane; idx < gg; idx += 32) {
        const int i = idx >> l, j = idx & (g - 1);
        const float tv = __ldg(Tl + idx);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int row = (i - ry[a]) & (g - 1);
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const float d = Db[a][b][row * g + ((j - rx[b]) & (g - 1))];
            acc[a][b] = fmaf(tv, d, acc[a][b]);
          }
        }
      }
    }
    const float wy1 = __int_as_float(pr.z), wx1 = __int_as_float(pr.w), wy0 = 1.f - wy1, wx0 = 1.f - wx1;
    float r = wy0 * (wx0 * acc[0][0] + wx1 * acc[0][1]) + wy1 * (wx0 * acc[1][0] + wx1 * acc[1][1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0) partial[v * units + unit] = r;
  }
}

__global__ void small_finish_kernel(const float* __restrict__ partial, const float* __restrict__ T,
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

template <int LOG2N>
hs_status launch_small_relight(const float* T, long long V, int faces, const float* planes, const int4* vparams,
                               float* partial, cudaStream_t st) {
  constexpr int SM = LOG2N * (1 << (2 * LOG2N)) * 4;
  HS_SMEM_ATTR(small_relight_kernel<LOG2N>, SM);
  const int units = 3 * faces;
  const int per_sm = (227 * 1024) / (SM + 1024) >= 2 ? 2 : 1;   // 2048 threads per SM at most
  int nsplit = sm_count() * per_sm / units;
  if (nsplit < 1) nsplit = 1;
  if (nsplit > V) nsplit = (int)V;
  small_relight_kernel<LOG2N><<<units * nsplit, kSWarps * 32, SM, st>>>(T, V, faces, planes, vparams, partial, nsplit);
  HS_CHECK_LAUNCH("small_relight_kernel");
  return HS_OK;
}

}  // namespace

size_t relight_small_planes_workspace_bytes(long long V, int faces, int log2n) {
  return (size_t)faces * 3 * log2n * ((size_t)1 << (2 * log2n)) * 4 + (size_t)V * 3 * faces * 4 + 256;
}

// N <= 64 (log2n <= 6): every level from residue planes
hs_status launch_relight_small_planes(const float* T, long long V, int faces, const float* light, int log2n,
                                      const double* fields64, long long face_stride, const int4* vparams, float* R,
                                      void* ws, cudaStream_t st) {
  if (log2n < 1 || log2n > 6) return HS_ERR_UNSUPPORTED;
  float* planes = reinterpret_cast<float*>(ws);
  float* partial = planes + (size_t)faces * 3 * log2n * ((size_t)1 << (2 * log2n));
  const int units = 3 * faces;
  const size_t psm = (size_t)2 * ((size_t)1 << (2 * log2n)) * 8;
  HS_SMEM_ATTR(small_planes_kernel, 2 * 4096 * 8);
  small_planes_kernel<<<units, 512, psm, st>>>(fields64, face_stride, log2n, planes);
  HS_CHECK_LAUNCH("small_planes_kernel");
  hs_status s = HS_OK;
  switch (log2n) {
    case 1: s = launch_small_relight<1>(T, V, faces, planes, vparams, partial, st); break;
    case 2: s = launch_small_relight<2>(T, V, faces, planes, vparams, partial, st); break;
    case 3: s = launch_small_relight<3>(T, V, faces, planes, vparams, partial, st); break;
    case 4: s = launch_small_relight<4>(T, V, faces, planes, vparams, partial, st); break;
    case 5: s = launch_small_relight<5>(T, V, faces, planes, vparams, partial, st); break;
    default: s = launch_small_relight<6>(T, V, faces, planes, vparams, partial, st); break;
  }
  if (s != HS_OK) return s;
  small_finish_kernel<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(partial, T, light, V, faces, log2n, R);
  HS_CHECK_LAUNCH("small_finish_kernel");
  return HS_OK;
}

namespace {
}  // namespace

size_t relight_planes_workspace_bytes(long long V, int faces) {
  return (size_t)faces * 3 * kPlanesPerUnit * 4 + (size_t)V * 6 * faces * 4 + 256;
}

// fields64: fp64 level-n fields of face f at fields64 + f * face_stride, [3][N][N]
hs_status launch_relight_planes(const float* T, long long V, int faces, const float* light, const double* fields64,
                                long long face_stride, const int4* vparams, float* R, void* ws, cudaStream_t st) {
  float* planes = reinterpret_cast<float*>(ws);
  float* partial = planes + (size_t)faces * 3 * kPlanesPerUnit;
  const int units = 3 * faces;
  HS_SMEM_ATTR(planes_kernel, 4 * 4096 * 8);
  HS_SMEM_ATTR(planes_a_kernel, kASmem);
  HS_SMEM_ATTR(planes_c_kernel, kCSmem);
  planes_kernel<<<units, 512, 4 * 4096 * 8, st>>>(fields64, face_stride, planes);
  HS_CHECK_LAUNCH("planes_kernel");
  planes3_kernel<<<units, 256, 0, st>>>(planes);
  HS_CHECK_LAUNCH("planes3_kernel");
  HS_SMEM_ATTR(planes_low_kernel, 2 * kPL * 4);
  planes_low_kernel<<<units, 512, 2 * kPL * 4, st>>>(planes);
  HS_CHECK_LAUNCH("planes_low_kernel");
  int nsplit = sm_count() / units;
  if (nsplit < 1) nsplit = 1;
  if (nsplit > V) nsplit = (int)V;
  planes_a_kernel<<<units * nsplit, kAWarps * 32, kASmem, st>>>(T, V, faces, planes, vparams, partial, nsplit);
  HS_CHECK_LAUNCH("planes_a_kernel");
  planes_c_kernel<<<units * nsplit, kCWarps * 32, kCSmem, st>>>(T, V, faces, planes, vparams, partial, nsplit);
  HS_CHECK_LAUNCH("planes_c_kernel");
  planes_finish_kernel<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(partial, T, light, V, faces, R);
  HS_CHECK_LAUNCH("planes_finish_kernel");
  return HS_OK;
}

}  // namespace hs
