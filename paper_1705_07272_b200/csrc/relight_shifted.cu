// Fused per-vertex shift + relight:  r_v = < S_{s_v} L , T_v >
// (every pixel/vertex rotates by its own normal angles; the coarser levels
// follow by the recursive h_s / h_t filters; plugged into the light-transport integral).
// DESIGN.md §5.5.
//
// The shifted pyramid of a vertex is never materialised.  Per call:
//   fields_kernel         the light's full-resolution difference fields F_n (fp64, once: the light
//                         is shared by all vertices);
//   vertex_params_kernel  each vertex's shift split into (q, phi) in fp64 (row a0);
//   residue planes        (csrc/relight_planes.cu) the box shift is four integer rolls of F_n and
//                         the bottom-up commutes with even rolls, so every output level is a rolled
//                         read of planes precomputed from the light over the shift residues: per
//                         vertex only dot products remain.  N <= 64: every level from planes; N = 128:
//                         levels n-1 .. n-3 from planes, the last four by the warp's own bottom-up.
// Larger faces take the chunked path in abi.cu (batched tile shift + row dot).
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// The full-resolution difference fields F_n (X, Y, Z) of every face of the light, top-down from its
// detail coefficients only, one CTA per face, level by level,
// in fp64 (an fp32 recursion carries an absolute error ~eps |A| at pixel-value scale, ~1e4 for HDR
// suns, into every difference).  Level l+1 lands in scratch + f 6 N^2 + ((l+1) & 1) 3 N^2, natural
// layout [3][2^(l+1)][2^(l+1)]; the final level is what the residue planes are built from.
__global__ void __launch_bounds__(kThreads) fields_kernel(const float* __restrict__ light, int n,
                                                          double* __restrict__ scratch) {
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
          const int o = (2 * i + a) * G + (2 * j + b);
          nxt[o] = cx[a][b];
          nxt[G * G + o] = cy[a][b];
          nxt[2 * G * G + o] = cz[a][b];
        }
    }
    __syncthreads();
    __threadfence_block();
  }
}

// ------------------------------------------------------------------------------- main
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

}  // namespace

bool relight_shifted_fused_supported(int log2n) { return log2n >= 1 && log2n <= 7; }

size_t relight_shifted_fused_workspace_bytes(long long V, int faces, int log2n) {
  const size_t NN = (size_t)1 << (2 * log2n);
  return (size_t)faces * 6 * NN * 8 /*fp64 fields, ping-pong*/ + (size_t)V * 16 /*vertex params*/ + 512 +
         (log2n == 7 ? relight_planes_workspace_bytes(V, faces) : relight_small_planes_workspace_bytes(V, faces, log2n));
}

hs_status launch_relight_shifted_fused(const float* T, long long V, int faces, const float* light, int log2n,
                                       const float* shifts, float* R, void* ws, cudaStream_t st) {
  if (!relight_shifted_fused_supported(log2n)) return HS_ERR_UNSUPPORTED;
  const size_t NN = (size_t)1 << (2 * log2n);
  double* scratch = reinterpret_cast<double*>(ws);
  int4* vp = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(scratch + (size_t)faces * 6 * NN) + 255) &
                                     ~uintptr_t(255));
  void* pws = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(vp + V) + 255) & ~uintptr_t(255));
  fields_kernel<<<faces, kThreads, 0, st>>>(light, log2n, scratch);
  HS_CHECK_LAUNCH("fields_kernel");
  vertex_params_kernel<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(shifts, V, 1 << log2n, vp);
  HS_CHECK_LAUNCH("vertex_params_kernel");
  const double* fields64 = scratch + (log2n & 1) * 3 * NN;   // fields_kernel's last level
  if (log2n == 7) return launch_relight_planes(T, V, faces, light, fields64, (long long)(6 * NN), vp, R, pws, st);
  return launch_relight_small_planes(T, V, faces, light, log2n, fields64, (long long)(6 * NN), vp, R, pws, st);
}

}  // namespace hs
