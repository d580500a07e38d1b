// Relight: R[v][b] = sum_f sum_{k<k_face} T[v][f k_face + k] L[b][f][k].
// The double product of PAPER.md eq:tripleSum with C_{ij0} = delta_ij (P:287,
// P:291-294), "plugged in the triple integral computation".  DESIGN.md §5.2.
//
//  * batch <= 8: streaming GEMV on CUDA cores.  HBM-bound: every T element is read once with
//    128-bit non-allocating loads; each warp owns RPW rows so a light float4 (L1/L2 resident) is
//    reused across RPW rows; per-row reduction order is fixed (independent of the row count and of
//    multi-GPU sharding).
//  * batches that are multiples of 64 (and K % 64 == 0): the tcgen05 split-precision kernel
//    (relight_tc.cu); other batches: CUDA-core tiled GEMM (128 rows x 64 frames x 32 k).
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

__device__ __forceinline__ float4 ld_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

template <int B, int RPW>
__global__ void __launch_bounds__(256) relight_gemv_kernel(const float* __restrict__ T, long long V, int K,
                                                           int kshift, const float* __restrict__ L,
                                                           long long lstride, long long lbatch,
                                                           float* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int kmask = (1 << kshift) - 1;
  for (long long r0 = warp * RPW; r0 < V; r0 += nwarps * RPW) {
    float acc[RPW][B];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int b = 0; b < B; ++b) acc[r][b] = 0.f;
    const float* Tr[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const long long row = (r0 + r < V) ? r0 + r : V - 1;
      Tr[r] = T + row * (long long)K;
    }
#pragma unroll 4
    for (int k = lane * 4; k < K; k += 128) {
      float4 t[RPW];
#pragma unroll
      for (int r = 0; r < RPW; ++r) t[r] = ld_stream(Tr[r] + k);
      const long long lo = (long long)(k >> kshift) * lstride + (k & kmask);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const float4 l = __ldg(reinterpret_cast<const float4*>(L + b * lbatch + lo));
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          acc[r][b] = fmaf(t[r].x, l.x, acc[r][b]);
          acc[r][b] = fmaf(t[r].y, l.y, acc[r][b]);
          acc[r][b] = fmaf(t[r].z, l.z, acc[r][b]);
          acc[r][b] = fmaf(t[r].w, l.w, acc[r][b]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float v = acc[r][b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[r][b] = v;
      }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < RPW; ++r)
        if (r0 + r < V)
#pragma unroll
          for (int b = 0; b < B; ++b) R[(r0 + r) * B + b] = acc[r][b];
    }
  }
}

// Short rows (K <= 4096, one frame): one row per 256-thread block, every thread's float4 loads
// issued at once -- a single HBM round trip per row instead of K / 512 dependent ones (the c2
// step is latency-bound).  Fixed reduction order (thread, warp tree, warps in order): per-row
// results depend on K only, not on the row count or the sharding.
constexpr int kShortK = 4096;
__global__ void __launch_bounds__(256) relight_gemv_short_kernel(const float* __restrict__ T, long long V, int K,
                                                                 int kshift, const float* __restrict__ L,
                                                                 long long lstride, float* __restrict__ R) {
  __shared__ float part[8];
  const int kmask = (1 << kshift) - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (long long row = blockIdx.x; row < V; row += gridDim.x) {
    const float* Tr = T + row * (long long)K;
    float4 t[kShortK / 1024], l[kShortK / 1024];
#pragma unroll
    for (int u = 0; u < kShortK / 1024; ++u) {
      const int k = (tid + u * 256) * 4;
      if (k < K) {
        t[u] = ld_stream(Tr + k);
        l[u] = __ldg(reinterpret_cast<const float4*>(L + (long long)(k >> kshift) * lstride + (k & kmask)));
      } else {
        t[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        l[u] = t[u];
      }
    }
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < kShortK / 1024; ++u) {
      acc = fmaf(t[u].x, l[u].x, acc);
      acc = fmaf(t[u].y, l[u].y, acc);
      acc = fmaf(t[u].z, l[u].z, acc);
      acc = fmaf(t[u].w, l[u].w, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      float sum = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) sum += part[w];
      R[row] = sum;
    }
    __syncthreads();
  }
}

constexpr int GM = 128, GN = 64, GK = 32;

__global__ void __launch_bounds__(256) relight_gemm_kernel(const float* __restrict__ T, long long V, int K,
                                                           int kshift, const float* __restrict__ L,
                                                           long long lstride, long long lbatch, int B,
                                                           float* __restrict__ R) {
  __shared__ __align__(16) float As[GK][GM + 4];
  __shared__ __align__(16) float Bs[GK][GN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const long long row0 = (long long)blockIdx.x * GM;
  const int b0 = blockIdx.y * GN;
  const int kmask = (1 << kshift) - 1;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += GK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * 256;
      const int row = idx >> 3, c4 = idx & 7;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row0 + row < V && k0 + c4 * 4 < K) v = ld_stream(T + (row0 + row) * (long long)K + k0 + c4 * 4);
      As[c4 * 4 + 0][row] = v.x;
      As[c4 * 4 + 1][row] = v.y;
      As[c4 * 4 + 2][row] = v.z;
      As[c4 * 4 + 3][row] = v.w;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * 256;
      const int b = idx >> 3, c4 = idx & 7;
      const int k = k0 + c4 * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b0 + b < B && k < K)
        v = __ldg(reinterpret_cast<const float4*>(L + (long long)(b0 + b) * lbatch +
                                                  (long long)(k >> kshift) * lstride + (k & kmask)));
      Bs[c4 * 4 + 0][b] = v.x;
      Bs[c4 * 4 + 1][b] = v.y;
      Bs[c4 * 4 + 2][b] = v.z;
      Bs[c4 * 4 + 3][b] = v.w;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long row = row0 + ty * 8 + i;
    if (row >= V) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = b0 + tx * 4 + j;
      if (b < B) R[row * B + b] = acc[i][j];
    }
  }
}

__global__ void __launch_bounds__(256) rowdot_kernel(const float* __restrict__ T, const float* __restrict__ S,
                                                     long long rows, long long K, float* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < rows; r += nwarps) {
    const float* t = T + r * K;
    const float* s = S + r * K;
    float acc = 0.f;
#pragma unroll 4
    for (long long k = lane * 4; k < K; k += 128) {
      const float4 a = ld_stream(t + k);
      const float4 b = __ldcg(reinterpret_cast<const float4*>(s + k));
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
      acc = fmaf(a.z, b.z, acc);
      acc = fmaf(a.w, b.w, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) R[r] = acc;
  }
}

int sm_count() { return device_sm_count(); }

template <int B, int RPW>
hs_status gemv_launch(const float* T, long long V, int K, int kshift, const float* L, long long lstride,
                      long long lbatch, float* R, int threads, cudaStream_t st) {
  const long long groups = (V + RPW - 1) / RPW;
  const int wpb = threads / 32;
  long long blocks = (groups + wpb - 1) / wpb;
  const long long cap = (long long)sm_count() * 2048 / threads;  // grid-stride beyond one full wave
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  relight_gemv_kernel<B, RPW><<<(unsigned)blocks, threads, 0, st>>>(T, V, K, kshift, L, lstride, lbatch, R);
  HS_CHECK_LAUNCH("relight_gemv_kernel");
  return HS_OK;
}

// Two-warp blocks: with ~2 rows per warp the block count is large enough for the block scheduler to
// balance the SMs dynamically (8-warp blocks left whole blocks of imbalance: 74 % vs 100 % of the
// copy peak at c3).
template <int B>
hs_status gemv(const float* T, long long V, int K, int kshift, const float* L, long long lstride,
               long long lbatch, float* R, cudaStream_t st) {
  return gemv_launch<B, (B <= 4) ? 2 : 1>(T, V, K, kshift, L, lstride, lbatch, R, 64, st);
}

}  // namespace

hs_status launch_relight_tc(const float* T, long long V, int faces, int kface, const float* L, long long lstride,
                            int batch, float* R, void* ws, size_t ws_bytes, cudaStream_t st, bool* handled);

hs_status launch_relight(const float* T, long long V, int faces, int kface, const float* L,
                         long long lstride, int batch, float* R, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int K = faces * kface;
  int kshift = 0;
  while ((1 << kshift) < kface) ++kshift;
  const long long lbatch = (long long)faces * lstride;
  if (batch == 1 && K <= kShortK) {
    long long blocks = V;
    const long long cap = (long long)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    relight_gemv_short_kernel<<<(unsigned)blocks, 256, 0, st>>>(T, V, K, kshift, L, lstride, R);
    HS_CHECK_LAUNCH("relight_gemv_short_kernel");
    return HS_OK;
  }
  switch (batch) {
    case 1: return gemv<1>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 2: return gemv<2>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 3: return gemv<3>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 4: return gemv<4>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 5: return gemv<5>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 6: return gemv<6>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 7: return gemv<7>(T, V, K, kshift, L, lstride, lbatch, R, st);
    case 8: return gemv<8>(T, V, K, kshift, L, lstride, lbatch, R, st);
    default: break;
  }
  bool handled = false;
  hs_status s = launch_relight_tc(T, V, faces, kface, L, lstride, batch, R, ws, ws_bytes, st, &handled);
  if (handled || s != HS_OK) return s;
  dim3 grid((unsigned)((V + GM - 1) / GM), (unsigned)((batch + GN - 1) / GN));
  relight_gemm_kernel<<<grid, 256, 0, st>>>(T, V, K, kshift, L, lstride, lbatch, batch, R);
  HS_CHECK_LAUNCH("relight_gemm_kernel");
  return HS_OK;
}

hs_status launch_rowdot(const float* T, const float* S, long long rows, long long K, float* R, cudaStream_t st) {
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  rowdot_kernel<<<(unsigned)blocks, 256, 0, st>>>(T, S, rows, K, R);
  HS_CHECK_LAUNCH("rowdot_kernel");
  return HS_OK;
}

}  // namespace hs
