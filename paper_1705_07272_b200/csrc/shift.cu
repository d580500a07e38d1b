// Host side of haar_shift_coeffs: shift classification (row a0), workspace layout, chunked
// launches; plus the 1D kernel (one CTA per signal, everything in shared memory).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace hs {

hs_status launch_shift2d(ShiftArgs& a, int max_tiles, bool any_coarse, bool any_perm, bool any_tile, int max_band_m,
                         cudaStream_t st);
int shift2d_tiles_for(int m);

namespace {

constexpr int k1DThreads = 256;

// 1D shift, one CTA per signal.  The paper's difference recursion
//   Delta_l[k] = a_l[k] - a_l[k+1]; top-down Delta_{l+1}[2k] = 2 d^_l[k],
//   Delta_{l+1}[2k+1] = Delta_l[k] - d^_l[k] - d^_l[k+1]; shift at level m;
//   bottom-up d^'_l[k] = Delta'_{l+1}[2k] / 2, Delta'_l[k] = (D'[2k] + 2 D'[2k+1] + D'[2k+2]) / 2
// is carried on its antiderivative a (as the 2D band kernel): a_0 = 0,
// a_{l+1}[2k] = a_l[k] + d^_l[k], a_{l+1}[2k+1] = a_l[k] - d^_l[k]; a' = w0 a[x - Q] + w1 a[x - Q - 1];
// d^'_l[k] = (a'[2k] - a'[2k+1]) / 2 (= Delta'[2k] / 2), a'_l[k] = (a'[2k] + a'[2k+1]) / 2 (whose
// difference is the [1,2,1] / 2 recursion above).  The signal's levels < m are staged into shared
// memory in one round trip (one global load per level made the kernel latency-bound: 60 us for
// 4096 signals of 4096); fp64 in shared memory (one rounding per output: fp32 rounding of the fine
// values is amplified ~2^(n-l) on a coarse band).
__global__ void __launch_bounds__(k1DThreads) shift1d_kernel(const __grid_constant__ ShiftArgs args) {
  extern __shared__ __align__(16) double smem[];
  const int g = blockIdx.x;
  const FaceParam P = args.dev_fp ? args.dev_fp[g] : args.fp[g];
  const int n = args.log2n;
  const int m = P.m;
  const int b = g / args.faces, f = g % args.faces;
  const float* __restrict__ in = args.in + (long long)b * args.in_batch_stride + (long long)f * args.in_face_stride;
  float* __restrict__ out = args.out + (long long)g * args.out_face_stride;
  const int band = args.band;
  const int Kb = 1 << band;
  const int gm = 1 << m;
  double* cur = smem;                                        // 2^m doubles
  double* nxt = smem + gm;                                   // 2^m doubles
  float* S = reinterpret_cast<float*>(smem + 2 * gm);        // in[0 .. 2^m): levels < m
  // levels >= m: permutation by q / 2^(n-l); scaling copied
  for (int idx = threadIdx.x; idx < Kb; idx += blockDim.x) {
    if (idx == 0) {
      out[0] = in[0];
      continue;
    }
    const int l = 31 - __clz(idx);
    if (l < m) continue;
    const int k = idx - (1 << l);
    const int sk = (k - (P.qx >> (n - l))) & ((1 << l) - 1);
    out[idx] = in[(1 << l) + sk];
  }
  if (m == 0) return;
  if ((reinterpret_cast<unsigned long long>(in) & 15) == 0 && gm >= 4) {
    for (int idx = threadIdx.x; idx < gm / 4; idx += blockDim.x)
      reinterpret_cast<float4*>(S)[idx] = __ldg(reinterpret_cast<const float4*>(in) + idx);
  } else {
    for (int idx = threadIdx.x; idx < gm; idx += blockDim.x) S[idx] = __ldg(in + idx);
  }
  if (threadIdx.x == 0) cur[0] = 0.0;   // a_0 = 0: the scaling coefficient drops out of every output
  __syncthreads();
  for (int l = 0; l < m; ++l) {
    const int gl = 1 << l;
    const double asc = exp2((double)l * 0.5);  // unit-interval -> averaging: x 2^(l/2)
    for (int kk = threadIdx.x; kk < gl; kk += blockDim.x) {
      const double a = cur[kk], d = (double)S[gl + kk] * asc;
      *reinterpret_cast<double2*>(nxt + 2 * kk) = make_double2(a + d, a - d);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  // shift at level m, then the analysis m-1 .. 0
  const double w0 = 1.0 - (double)P.wx, w1 = (double)P.wx;
  for (int x = threadIdx.x; x < gm; x += blockDim.x)
    nxt[x] = w0 * cur[(x - P.Qx) & (gm - 1)] + w1 * cur[(x - P.Qx - 1) & (gm - 1)];
  __syncthreads();
  {
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (int l = m - 1; l >= 0; --l) {
    const int gl = 1 << l;
    const double osc = exp2(-(double)l * 0.5);
    for (int kk = threadIdx.x; kk < gl; kk += blockDim.x) {
      const double2 a = *reinterpret_cast<const double2*>(cur + 2 * kk);
      nxt[kk] = 0.5 * (a.x + a.y);
      if (l < band) out[gl + kk] = (float)(0.5 * (a.x - a.y) * osc);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// Per-vertex shifts on the device (relight_vertices_shifted): the same fp64 classification.
__global__ void face_params_kernel(const float* __restrict__ shifts, long long num, int faces, int n,
                                   FaceParam* __restrict__ fp) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= num) return;
  const FaceParam p = make_face_param_2d((double)shifts[2 * v], (double)shifts[2 * v + 1], n);
  for (int f = 0; f < faces; ++f) fp[v * faces + f] = p;
}

}  // namespace

size_t shift_workspace_bytes_impl(int ndim, int log2n, long long num_faces) {
  if (ndim != 2) return 0;
  return (size_t)num_faces * (size_t)ws_face_floats_2d(log2n) * 8;
}

// in:  [num_faces / faces batches][faces][K]; out [num_faces][Kb]
hs_status launch_shift(const float* in, float* out, int ndim, int log2n, int faces,
                       long long num_faces, long long in_batch_stride, long long in_face_stride,
                       const double* shifts_host,
                       const float* shifts_dev_per_vertex, FaceParam* dev_fp_buf, int band,
                       void* ws, size_t ws_bytes, cudaStream_t st) {
  const int n = log2n;
  const long long Kb = (ndim == 2) ? (1ll << (2 * band)) : (1ll << band);
  float* wsf = nullptr;
  const long long wsface = (ndim == 2) ? ws_face_floats_2d(n) * 8 : 0;   // bytes per face
  if (ndim == 2) wsf = reinterpret_cast<float*>(ws);
  if (faces < 1 || faces > kMaxFacesPerLaunch) return HS_ERR_INVALID_ARG;   // ShiftArgs holds one chunk's faces
  const long long batches = num_faces / faces;
  const long long chunk_b = std::max<long long>(1, kMaxFacesPerLaunch / faces);
  ShiftArgs a;
  for (long long b0 = 0; b0 < batches; b0 += chunk_b) {
    const long long nb = std::min(chunk_b, batches - b0);
    const int nf = (int)(nb * faces);
    const long long g0 = b0 * faces;
    a.in = in + b0 * in_batch_stride;
    a.out = out + g0 * Kb;
    a.ws = wsf ? reinterpret_cast<float*>(reinterpret_cast<char*>(wsf) + g0 * wsface) : nullptr;
    a.dev_fp = nullptr;
    a.in_batch_stride = in_batch_stride;
    a.in_face_stride = in_face_stride;
    a.ws_face_stride = wsface;
    a.log2n = n;
    a.faces = faces;
    a.band = band;
    a.out_face_stride = (int)Kb;
    a.num_faces = nf;
    int max_tiles = 0;
    bool any_perm = false, any_coarse = false, any_tile = false;
    int max_band_m = 0;   // largest working level taken by the band kernel (0: none)
    a.band_path = (ndim == 2) ? 1 : 0;
    if (shifts_host) {
      for (int i = 0; i < nf; ++i) {
        const double* s = shifts_host + (g0 + i) * ndim;
        a.fp[i] = (ndim == 2) ? make_face_param_2d(s[0], s[1], n) : make_face_param_1d(s[0], n);
        max_tiles = std::max(max_tiles, shift2d_tiles_for(a.fp[i].m));
        if (a.fp[i].m < band || a.fp[i].m == 0) any_perm = true;
        if (a.band_path && band_level(a.fp[i].m)) {
          max_band_m = std::max(max_band_m, a.fp[i].m);
        } else if (a.fp[i].m > 0) {
          any_tile = true;
          if (coarse_level(a.fp[i].m) > 0) any_coarse = true;
        }
      }
    } else {
      // per-vertex device shifts: FaceParams computed on the device (one per vertex and face)
      FaceParam* dfp = dev_fp_buf + g0;
      const long long nv = nb;
      face_params_kernel<<<(unsigned)((nv + 127) / 128), 128, 0, st>>>(shifts_dev_per_vertex + b0 * 2, nv,
                                                                        faces, n, dfp);
      HS_CHECK_LAUNCH("face_params_kernel");
      a.dev_fp = dfp;
      max_tiles = shift2d_tiles_for(n);
      any_perm = true;
      any_coarse = coarse_level(n) > 0;
      any_tile = true;
      max_band_m = (a.band_path && n >= kBandMinLevel) ? std::min(n, kBandMaxLevel) : 0;
    }
    if (ndim == 2) {
      hs_status s = launch_shift2d(a, max_tiles, any_coarse, any_perm, any_tile, max_band_m, st);
      if (s != HS_OK) return s;
    } else {
      const size_t smem = (size_t)2 * (1u << n) * sizeof(double) + (size_t)(1u << n) * sizeof(float);
      if (smem > 48 * 1024) {
        HS_SMEM_ATTR(shift1d_kernel, smem);
      }
      shift1d_kernel<<<nf, k1DThreads, smem, st>>>(a);
      HS_CHECK_LAUNCH("shift1d_kernel");
    }
  }
  return HS_OK;
}

}  // namespace hs
