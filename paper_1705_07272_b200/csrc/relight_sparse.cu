// Sparse-transfer relight: every vertex keeps K_s (index, value) pairs of
// its transfer vector over the full-resolution pyramids (non-linear approximation, PAPER.md
// P:240-245), and the double product (eq:tripleSum with C_{ij0} = delta_ij) becomes a gather:
//   R[v][b] = sum_k val[v][k] * L[b][idx[v][k]].
// The light is transposed once per call to coefficient-major Lt[c][b] so that one index fetches
// the 64 frames of a coefficient as one contiguous 256-byte row (coalesced across the warp's
// lanes, which own the frames).  One warp per vertex; the warp loads 32 (index, value) pairs
// cooperatively and broadcasts them by shuffle.  Bound: L2 gather bandwidth (Lt is L2-resident);
// HBM traffic is only K_s * 8 bytes per vertex plus the radiance.  DESIGN.md §5.7.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

__host__ __device__ inline uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Mirror of synth.sparse_transfer_rows (bit for bit).
__global__ void fill_sparse_kernel(int* __restrict__ idx, float* __restrict__ val, long long row_start,
                                   long long rows, int faces, int n, int ks, int dense_levels, uint64_t base_ts,
                                   uint64_t base_t) {
  const long long total = rows * ks;
  const int nd = faces << (2 * dense_levels);
  const int nlev = (n - dense_levels) > 0 ? (n - dense_levels) : 1;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / ks;
    const int k = (int)(e - r * ks);
    const uint64_t gi = (uint64_t)(row_start + r) * (uint64_t)ks + (uint64_t)k;
    int f, coef;
    if (k < nd) {
      f = k >> (2 * dense_levels);
      coef = k & ((1 << (2 * dense_levels)) - 1);
    } else {
      const uint64_t h = smix(base_ts + gi);
      const int lev = dense_levels + (int)((h >> 8) % (uint64_t)nlev);
      const int typ = (int)((h >> 16) % 3ull);
      f = (int)((h >> 24) % (uint64_t)faces);
      const long long cell = (long long)((h >> 32) & 0xFFFFFFFFull) % (1ll << (2 * lev));
      coef = (int)((1ll << (2 * lev)) * (1 + typ) + cell);
    }
    idx[e] = f * (1 << (2 * n)) + coef;
    const uint64_t hu = smix(base_t + gi);
    float u = (float)((int)(hu >> 40) - (1 << 23)) * (1.0f / 8388608.0f);
    const int lvl = (coef == 0) ? 0 : ((31 - __clz(coef)) >> 1);
    u = ldexpf(u, -lvl);
    if (coef == 0) u = fabsf(u);
    val[e] = u;
  }
}

// L [B][C] -> Lt [C][B] (32 x 32 smem tiles)
__global__ void transpose_kernel(const float* __restrict__ L, long long C, int B, float* __restrict__ Lt) {
  __shared__ float tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int b0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int b = b0 + r;
    const long long c = c0 + threadIdx.x;
    tile[r][threadIdx.x] = (b < B && c < C) ? __ldg(L + (long long)b * C + c) : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const long long c = c0 + r;
    const int b = b0 + threadIdx.x;
    if (c < C && b < B) Lt[c * B + b] = tile[threadIdx.x][r];
  }
}

// One warp per vertex; lane owns frames b0 + lane and b0 + 32 + lane of the current frame block.
__global__ void __launch_bounds__(256) relight_sparse_kernel(const int* __restrict__ idx, const float* __restrict__ val,
                                                             long long V, int ks, const float* __restrict__ Lt, int B,
                                                             int b0, int bw, float* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const bool has0 = lane < bw, has1 = lane + 32 < bw;
  for (long long v = warp; v < V; v += nwarps) {
    const int* iv = idx + v * ks;
    const float* vv = val + v * ks;
    float a0 = 0.f, a1 = 0.f;
    for (int k0 = 0; k0 < ks; k0 += 32) {
      const int kk = k0 + lane;
      const int mi = kk < ks ? __ldg(iv + kk) : 0;
      const float mv = kk < ks ? __ldg(vv + kk) : 0.f;
      const int cnt = (ks - k0) < 32 ? (ks - k0) : 32;
#pragma unroll 8
      for (int j = 0; j < cnt; ++j) {
        const int i = __shfl_sync(0xffffffffu, mi, j);
        const float w = __shfl_sync(0xffffffffu, mv, j);
        const float* row = Lt + (long long)i * B + b0;
        if (has0) a0 = fmaf(w, __ldg(row + lane), a0);
        if (has1) a1 = fmaf(w, __ldg(row + 32 + lane), a1);
      }
    }
    if (has0) R[v * B + b0 + lane] = a0;
    if (has1) R[v * B + b0 + 32 + lane] = a1;
  }
}

// Full 64-frame blocks with K_s % 4 == 0: lane owns frames 2 lane, 2 lane + 1 (one 8-byte load per
// gathered row and lane: the warp's 256-byte row in one request), and the (index, value) pairs are
// read four at a time by every lane from the same address (a broadcast, no shuffles): ~4
// instructions per gathered entry instead of ~10.
__global__ void __launch_bounds__(256) relight_sparse64_kernel(const int* __restrict__ idx,
                                                               const float* __restrict__ val, long long V, int ks,
                                                               const float* __restrict__ Lt, int B, int b0,
                                                               float* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const float* base = Lt + b0 + 2 * lane;
  for (long long v = warp; v < V; v += nwarps) {
    const int4* iv = reinterpret_cast<const int4*>(idx + v * ks);
    const float4* vv = reinterpret_cast<const float4*>(val + v * ks);
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
    for (int k = 0; k < ks / 4; ++k) {
      const int4 i = __ldg(iv + k);
      const float4 w = __ldg(vv + k);
      const float2 x0 = __ldg(reinterpret_cast<const float2*>(base + (long long)i.x * B));
      const float2 x1 = __ldg(reinterpret_cast<const float2*>(base + (long long)i.y * B));
      const float2 x2 = __ldg(reinterpret_cast<const float2*>(base + (long long)i.z * B));
      const float2 x3 = __ldg(reinterpret_cast<const float2*>(base + (long long)i.w * B));
      a0 = fmaf(w.x, x0.x, a0);
      a1 = fmaf(w.x, x0.y, a1);
      a0 = fmaf(w.y, x1.x, a0);
      a1 = fmaf(w.y, x1.y, a1);
      a0 = fmaf(w.z, x2.x, a0);
      a1 = fmaf(w.z, x2.y, a1);
      a0 = fmaf(w.w, x3.x, a0);
      a1 = fmaf(w.w, x3.y, a1);
    }
    *reinterpret_cast<float2*>(R + v * B + b0 + 2 * lane) = make_float2(a0, a1);
  }
}

int sms() { return device_sm_count(); }

}  // namespace

hs_status launch_fill_sparse(int* idx, float* val, long long row_start, long long rows, int faces, int n, int ks,
                             int dense_levels, uint64_t seed, cudaStream_t st) {
  const uint64_t base_ts = smix(seed + 0x5A12ull * 0xD1B54A32D192ED03ull);
  const uint64_t base_t = smix(seed + 0x7A11ull * 0xD1B54A32D192ED03ull);
  long long blocks = (rows * ks + 255) / 256;
  if (blocks > (long long)sms() * 16) blocks = (long long)sms() * 16;
  if (blocks < 1) blocks = 1;
  fill_sparse_kernel<<<(unsigned)blocks, 256, 0, st>>>(idx, val, row_start, rows, faces, n, ks, dense_levels, base_ts,
                                                       base_t);
  HS_CHECK_LAUNCH("fill_sparse_kernel");
  return HS_OK;
}

hs_status launch_relight_sparse(const int* idx, const float* val, long long V, int ks, const float* light, long long C,
                                int B, float* R, float* Lt, cudaStream_t st) {
  dim3 tg((unsigned)((C + 31) / 32), (unsigned)((B + 31) / 32));
  transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(light, C, B, Lt);
  HS_CHECK_LAUNCH("transpose_kernel");
  long long blocks = (V + 7) / 8;
  if (blocks > (long long)sms() * 32) blocks = (long long)sms() * 32;
  if (blocks < 1) blocks = 1;
  // the vectorised kernel needs 16-byte (index, value) rows, 8-byte light rows and a full block
  const bool vec = (ks % 4 == 0) && (B % 2 == 0) && ((reinterpret_cast<uintptr_t>(R) & 7) == 0);
  for (int b0 = 0; b0 < B; b0 += 64) {
    const int bw = (B - b0) < 64 ? (B - b0) : 64;
    if (vec && bw == 64) {
      relight_sparse64_kernel<<<(unsigned)blocks, 256, 0, st>>>(idx, val, V, ks, Lt, B, b0, R);
      HS_CHECK_LAUNCH("relight_sparse64_kernel");
    } else {
      relight_sparse_kernel<<<(unsigned)blocks, 256, 0, st>>>(idx, val, V, ks, Lt, B, b0, bw, R);
      HS_CHECK_LAUNCH("relight_sparse_kernel");
    }
  }
  return HS_OK;
}

}  // namespace hs
