// Seeded transfer-matrix generator (input generation, not part of the method).  Bit-identical
// to synth.transfer_rows: a counter-based SplitMix64 hash of the global element
// index, so any row range of a tens-of-GB matrix is generated in place and the oracle
// regenerates any subset on the host.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {

__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_transfer_kernel(float* __restrict__ out, long long row_start, long long rows, int kt,
                                     int kshift, uint64_t base) {
  const long long total = rows * (long long)kt;
  const int kmask = (1 << kshift) - 1;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long v = e / kt;
    const int col = (int)(e - v * kt);
    const uint64_t gidx = (uint64_t)(row_start + v) * (uint64_t)kt + (uint64_t)col;
    const uint64_t h = splitmix64(base + gidx);
    const int u24 = (int)(h >> 40);
    float u = (float)(u24 - (1 << 23)) * (1.0f / 8388608.0f);
    const int k = col & kmask;
    const int lev = (k == 0) ? 0 : ((31 - __clz(k)) >> 1);
    u = ldexpf(u, -lev);
    if (k == 0) u = fabsf(u);
    out[e] = u;
  }
}

}  // namespace

hs_status launch_fill_transfer(float* out, long long row_start, long long rows, int faces, int kface,
                               uint64_t seed, uint64_t stream_id, cudaStream_t st) {
  int kshift = 0;
  while ((1 << kshift) < kface) ++kshift;
  const uint64_t base = splitmix64(seed + stream_id * 0xD1B54A32D192ED03ull);
  const long long total = rows * (long long)faces * kface;
  long long blocks = (total + 255) / 256;
  if (blocks > 148ll * 16) blocks = 148ll * 16;
  if (blocks < 1) blocks = 1;
  fill_transfer_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, row_start, rows, faces * kface, kshift, base);
  HS_CHECK_LAUNCH("fill_transfer_kernel");
  return HS_OK;
}

}  // namespace hs
