// tcgen05 / TMA / mbarrier PTX wrappers and host helpers shared by the tensor-core kernels
// (relight_tc.cu, relight_triple.cu).  Internal to libhaarshift.so.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <mutex>

namespace hs {
int device_sm_count();   // common.cuh: SMs of the current device, cached per device
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, 128-byte swizzle (8-row groups 1024 B apart).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major) = 1
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO = 1024 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// instruction descriptor: D f32, A/B f16, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_f16(int n, int m = 128) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// ------------------------------------------------------------------------------- host helpers
inline PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

inline int num_sms() { return ::hs::device_sm_count(); }

// (v - h) * 2^11 for a pair, as two packed f32x2 instructions (sm_100 FADD2 / FMUL2): the same
// roundings as the scalar form (the difference is exact, the power-of-two scale is exact)
__device__ __forceinline__ float2 resid2048(float2 v, float2 h) {
  float2 r;
  asm("{\n\t.reg .b64 va, ha, d, k;\n\tmov.b64 va, {%2, %3};\n\tmov.b64 ha, {%4, %5};\n\t"
      "mov.b64 k, {%6, %6};\n\tsub.rn.f32x2 d, va, ha;\n\tmul.rn.f32x2 d, d, k;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(v.x), "f"(v.y), "f"(h.x), "f"(h.y), "f"(2048.f));
  return r;
}


// ------------------------------------------------------------------------------- range handling
// Per-row power-of-two exponents of the split-precision tensor-core relights.
// The converter thread that owns a row picks e_v from the row's FIRST NONZERO 64-k block (in the
// common case block 0: one max over 64 values per row and tile) and splits every block of the row
// as x 2^e_v = hi + 2^-11 lo.  e_v = 0 while that block's max |x| lies in [2^-4, 2^8) -- then no
// scaling instruction runs at all -- else the scaled max lands in [2^7, 2^8).  Either way the split
// of every value is relative to the value itself for the 2^22 binades below the block's max, and
// the other blocks of the row may be up to 2^8 times larger before x 2^e_v leaves fp16's range.
// A row that does (|x 2^e_v| >= 65520: fp16 overflow) ends with a non-finite accumulator; the
// epilogue lists it and relight_redo_rows_kernel recomputes it exactly on the CUDA cores (fp64
// accumulation).  Every row's arithmetic depends on its own data only, so results do not depend on
// which rows share a tile (sharding is bitwise exact).  The epilogue multiplies by 2^-e_v, passed
// per (tile, row) through a ring of kExpRing int8 slots.
constexpr int kExpRing = 8;
__device__ __forceinline__ int row_exponent(float mx) {   // mx > 0, finite
  const int ex = ilogbf(mx);
  if (ex >= -4 && ex <= 7) return 0;
  const int e = 7 - ex;
  return e < -126 ? -126 : (e > 126 ? 126 : e);
}
__device__ __forceinline__ float pow2i(int e) { return __int_as_float((127 + e) << 23); }   // e in [-126, 127]
// fp16 hi / lo pieces of (a, b), lo = (x - hi) 2^11
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const float2 r = resid2048(make_float2(a, b), hf);
  const __half2 l = __floats2half2_rn(r.x, r.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// the same for (a, b) * sc (sc a power of two: the scaling is exact)
__device__ __forceinline__ void split_pair_scaled(float a, float b, float sc, uint32_t& hi, uint32_t& lo) {
  float2 v;
  asm("{\n\t.reg .b64 va, k;\n\tmov.b64 va, {%2, %3};\n\tmov.b64 k, {%4, %4};\n\t"
      "mul.rn.f32x2 va, va, k;\n\tmov.b64 {%0, %1}, va;\n\t}"
      : "=f"(v.x), "=f"(v.y)
      : "f"(a), "f"(b), "f"(sc));
  split_pair(v.x, v.y, hi, lo);
}
// Converter-side row exponent state: call at every k block (uniform control flow per warp).
struct RowExp {
  int e = 0;
  bool set = false, all_set = false, scaled = false;
  // kb == 0 resets; while any row of the warp is unset, `block_max()` is evaluated (warp-uniform).
  template <class MAXF>
  __device__ __forceinline__ void update(int kb, MAXF block_max) {
    if (kb == 0) {
      set = false;
      all_set = false;
      e = 0;
    }
    if (!all_set) {
      const float mx = block_max();
      if (!set && mx > 0.f && isfinite(mx)) {   // zero / non-finite blocks leave the row unset
        e = row_exponent(mx);
        set = true;
      }
      all_set = __all_sync(0xffffffffu, set);
      scaled = __any_sync(0xffffffffu, e != 0);
    }
  }
};
// Rows whose result came out non-finite (epilogue -> relight_redo_rows_kernel), in the workspace.
constexpr int kRedoCap = 8192;
struct RedoList {
  int count;
  int pad[3];
  long long rows[kRedoCap];
};
__device__ __forceinline__ void redo_push(RedoList* rl, long long row) {
  const int i = atomicAdd(&rl->count, 1);
  if (i < kRedoCap) rl->rows[i] = row;
}

// Exact recomputation of the listed rows on the CUDA cores: R[v][b] = sum_k x_v[k] L[b][k] with
// fp64 accumulation, x_v produced in shared-memory chunks by `fill` (the transfer row itself, or the
// tripling terms of relight_triple.cu).  L[b][k] = L[b * lbstride + (k >> kshift) * lstride +
// (k & (2^kshift - 1))].  One CTA of 128 threads per row; if more rows than kRedoCap were listed,
// every row whose radiance holds a non-finite value is recomputed instead (a scan of R).
constexpr int kRedoChunk = 2048;
template <class FILL>
__global__ void __launch_bounds__(128) relight_redo_rows_kernel(FILL fill, const float* __restrict__ L,
                                                                long long lbstride, long long lstride, int kshift,
                                                                int K, int B, float* __restrict__ R, long long V,
                                                                const RedoList* __restrict__ rl) {
  __shared__ float sx[kRedoChunk];
  __shared__ int sbad;
  const int cnt = rl->count;
  if (cnt == 0) return;
  const bool scan = cnt > kRedoCap;
  const long long n = scan ? V : cnt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long kmask = (1ll << kshift) - 1;
  for (long long e = blockIdx.x; e < n; e += gridDim.x) {
    const long long row = scan ? e : rl->rows[e];
    if (scan) {
      if (threadIdx.x == 0) sbad = 0;
      __syncthreads();
      for (int b = threadIdx.x; b < B; b += blockDim.x)
        if (!isfinite(R[row * B + b])) sbad = 1;
      __syncthreads();
      const int bad = sbad;
      __syncthreads();
      if (!bad) continue;
    }
    for (int fb0 = 0; fb0 < B; fb0 += 64) {
      double acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = 0.0;
      for (int k0 = 0; k0 < K; k0 += kRedoChunk) {
        const int nk = (K - k0) < kRedoChunk ? (K - k0) : kRedoChunk;
        __syncthreads();
        fill(row, k0, nk, sx);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int b = fb0 + warp * 16 + i;
          const float* Lb = L + (long long)b * lbstride;
          double a = acc[i];
          for (int k = lane; k < nk; k += 32) {
            const long long kk = k0 + k;
            a = fma((double)sx[k], (double)__ldg(Lb + (kk >> kshift) * lstride + (kk & kmask)), a);
          }
          acc[i] = a;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        double a = acc[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) R[row * B + fb0 + warp * 16 + i] = (float)a;
      }
    }
  }
}

}  // namespace tc
}  // namespace hs
