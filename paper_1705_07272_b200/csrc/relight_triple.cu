// Triple-product relight: BRDF and visibility kept separate,
//   R[v][b] = sum_f  integral of  L'_bf * rho_vf * V_vf        (eq:tripleSum)
// evaluated with the Tripling Coefficient Theorem in O(K) per (vertex, frame) block and
// fed to the 5th-generation tensor cores as a GEMM against the light.
//
// Layout ("qtree", include/haarshift.h haar_pack_qtree): a face of K_face = 4^k coefficients
// (k >= 3) is 4^r chunks of 64 floats, r = k - 3, one per level-r cell c (row-major); chunk c holds
// the 63 detail coefficients of the 3-level subtree under c (levels r, r+1, r+2) in post-order and,
// in slot 63, the mean of the function over cell c (the level-r approximation, which carries the
// same information as the coarse pyramid levels < r).
//
// Per chunk, with cell means A (top-down inside the subtree, from the slot-63 mean), pair sums
// P_n = sum_t rho_t V_t per node n, subtree sums S_n = P_n + sum of S over n's children, and
// the wavelet amplitude w_l = 2^l (unit-square normalisation):
//   M_t(n) = V_t A_rho(n) + rho_t A_V(n)                     case (c): pair (L, V) or (L, rho),
//                                                             third = scaling + coarser wavelets
//          + w_l (rho_t' V_t'' + rho_t'' V_t')               case (b): three distinct types
//          + w_l sum_q sign_t(q) S(child q)                   case (c): pair (rho, V) below n,
//                                                             third = L's wavelet at n
//   slot 63: 4^-r A_rho(c) A_V(c) + S(c)                      paired with the light's mean over c
// so that  R[v][b] = sum_chunks sum_s M[v][s] * Lq[b][s]  with Lq = the light packed the same way.
// The oracle (oracle/relight.py relight_triple) integrates the product of the three functions
// pixel by pixel instead; the two share nothing.
//
// Kernels:
//   pack_qtree_kernel      HAAR1 -> qtree (a permutation + the level-r cell means)
//   triple_text_kernel     CUDA-core fallback: M materialised per row chunk, then relight_vertices
//   relight_triple_tc_kernel  persistent, one CTA per SM, 12 warps:
//     warp 0  TMA producer of the rho and V tiles [128 rows x 64] (128B-swizzled, 3 stages)
//     warp 3  bulk-copy producer of the pre-split light tiles (2 stages)
//     warp 1  MMA issuer (tcgen05.mma kind::f16, A from TMEM) -- as in relight_tc.cu
//     warp 2  TMEM allocator
//     warps 4-7  converters: evaluate the tripling terms of their row's chunk from smem, scale
//                them by the row's power of two 2^e (tc_ptx.cuh RowExp), split fp32 -> fp16 hi/lo,
//                tcgen05.st into the A stage -- M never touches HBM
//     warps 8-11 epilogue: drains every KG = 16 k blocks into fp32 registers, scales by 2^-e and
//                the per-frame scale, lists non-finite rows for the exact CUDA-core redo
//                (relight_redo_rows_kernel), as in relight_tc.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace hs {
namespace {
using namespace tc;

constexpr int QC = 64;            // slots per qtree chunk

// wavelet signs on quadrant q = 2a + b (a: lower-half row bit, b: right-half column bit):
// H + on the left half, V + on the top half, D + on the main diagonal
__host__ __device__ constexpr float sgn_h(int q) { return (q & 1) ? -1.f : 1.f; }
__host__ __device__ constexpr float sgn_v(int q) { return (q & 2) ? -1.f : 1.f; }
__host__ __device__ constexpr float sgn_d(int q) { return (((q >> 1) ^ q) & 1) ? -1.f : 1.f; }

__device__ __forceinline__ float comp(const float4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// One node: M_t without the children fold, and the pair sum P.
__device__ __forceinline__ void node_terms(const float* x, const float* y, float Ax, float Ay, float w, float* M,
                                           float& P) {
  M[0] = fmaf(y[0], Ax, fmaf(x[0], Ay, w * fmaf(x[1], y[2], x[2] * y[1])));
  M[1] = fmaf(y[1], Ax, fmaf(x[1], Ay, w * fmaf(x[0], y[2], x[2] * y[0])));
  M[2] = fmaf(y[2], Ax, fmaf(x[2], Ay, w * fmaf(x[0], y[1], x[1] * y[0])));
  P = fmaf(x[0], y[0], fmaf(x[1], y[1], x[2] * y[2]));
}

// Slots 15q .. 15q+14 (child group q: four grandchildren, then the child) of one chunk.
template <class LD>
__device__ __forceinline__ void load_group(LD ld, int q, float* g) {
  const int s0 = 15 * q, u0 = s0 >> 2;
  float4 U[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) U[i] = ld(u0 + i);
#pragma unroll
  for (int i = 0; i < 15; ++i) g[i] = comp(U[((s0 + i) >> 2) - u0], (s0 + i) & 3);
}

// The 64 GEMM coefficients of one qtree chunk from the chunk of rho and of V.
// ld_r(u), ld_v(u): the 16-byte unit u (slots 4u .. 4u+3) of the chunk.
template <class LDR, class LDV>
__device__ __forceinline__ void triple_chunk(LDR ld_r, LDV ld_v, float w0, float inv_cells, float* out) {
  const float4 rr = ld_r(15), vv = ld_v(15);
  const float rx[3] = {rr.x, rr.y, rr.z}, vx[3] = {vv.x, vv.y, vv.z};
  const float Ar0 = rr.w, Av0 = vv.w;
  const float w1 = 2.f * w0, w2 = 4.f * w0;
  float fold0[3] = {0.f, 0.f, 0.f}, S0 = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float gr[15], gv[15];
    load_group(ld_r, q, gr);
    load_group(ld_v, q, gv);
    const float Ar1 = fmaf(w0, sgn_h(q) * rx[0] + sgn_v(q) * rx[1] + sgn_d(q) * rx[2], Ar0);
    const float Av1 = fmaf(w0, sgn_h(q) * vx[0] + sgn_v(q) * vx[1] + sgn_d(q) * vx[2], Av0);
    const float* cr = gr + 12;
    const float* cv = gv + 12;
    float fold1[3] = {0.f, 0.f, 0.f}, S1 = 0.f;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float Ar2 = fmaf(w1, sgn_h(p) * cr[0] + sgn_v(p) * cr[1] + sgn_d(p) * cr[2], Ar1);
      const float Av2 = fmaf(w1, sgn_h(p) * cv[0] + sgn_v(p) * cv[1] + sgn_d(p) * cv[2], Av1);
      float P2;
      node_terms(gr + 3 * p, gv + 3 * p, Ar2, Av2, w2, out + 15 * q + 3 * p, P2);
      S1 += P2;
      fold1[0] = fmaf(sgn_h(p), P2, fold1[0]);
      fold1[1] = fmaf(sgn_v(p), P2, fold1[1]);
      fold1[2] = fmaf(sgn_d(p), P2, fold1[2]);
    }
    float M1[3], P1;
    node_terms(cr, cv, Ar1, Av1, w1, M1, P1);
#pragma unroll
    for (int t = 0; t < 3; ++t) out[15 * q + 12 + t] = fmaf(w1, fold1[t], M1[t]);
    S1 += P1;
    S0 += S1;
    fold0[0] = fmaf(sgn_h(q), S1, fold0[0]);
    fold0[1] = fmaf(sgn_v(q), S1, fold0[1]);
    fold0[2] = fmaf(sgn_d(q), S1, fold0[2]);
  }
  float M0[3], P0;
  node_terms(rx, vx, Ar0, Av0, w0, M0, P0);
#pragma unroll
  for (int t = 0; t < 3; ++t) out[60 + t] = fmaf(w0, fold0[t], M0[t]);
  out[63] = fmaf(inv_cells * Ar0, Av0, S0 + P0);
}

// ------------------------------------------------------------------------------- packing
// out[row][f][c*64 + s] from in[row*faces*in_face_stride + f*in_face_stride + HAAR1 index]
// One thread per output slot: grid.x over the 4^k slots of one face band, grid.y = row * faces + f.
// (A flat grid-stride form with 64-bit index math ran at 0.3 TB/s: 102 us for 4096 BRDF rows.)
__global__ void __launch_bounds__(256) pack_qtree_kernel(const float* __restrict__ in, int faces,
                                                         long long in_face_stride, int k, float* __restrict__ out) {
  const int r = k - 3;
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= (1 << (2 * k))) return;
  const long long rf = blockIdx.y + (long long)blockIdx.z * gridDim.y;   // row * faces + f
  const float* src = in + rf * in_face_stride;
  const int c = pos >> 6, s = pos & 63;
  const int ci = c >> r, cj = c & ((1 << r) - 1);
  float v;
  if (s == 63) {
    float a = __ldg(src);
    for (int l = 0; l < r; ++l) {
      const int ai = ci >> (r - l), aj = cj >> (r - l);
      const int q = (((ci >> (r - l - 1)) & 1) << 1) | ((cj >> (r - l - 1)) & 1);
      const int base = (1 << (2 * l)), cell = ai * (1 << l) + aj;
      const float h = __ldg(src + base + cell), vv = __ldg(src + 2 * base + cell), d = __ldg(src + 3 * base + cell);
      a = fmaf(ldexpf(1.f, l), sgn_h(q) * h + sgn_v(q) * vv + sgn_d(q) * d, a);
    }
    v = a;
  } else {
    int l, t, i, j;
    if (s >= 60) {
      l = r, t = s - 60, i = ci, j = cj;
    } else {
      const int q = s / 15, u = s - 15 * q;
      const int i1 = 2 * ci + (q >> 1), j1 = 2 * cj + (q & 1);
      if (u >= 12) {
        l = r + 1, t = u - 12, i = i1, j = j1;
      } else {
        const int p = u / 3;
        l = r + 2, t = u - 3 * p, i = 2 * i1 + (p >> 1), j = 2 * j1 + (p & 1);
      }
    }
    v = __ldg(src + (1 << (2 * l)) * (1 + t) + i * (1 << l) + j);
  }
  out[(rf << (2 * k)) + pos] = v;
}

// ------------------------------------------------------------------------------- CUDA-core fallback
__global__ void __launch_bounds__(128) triple_text_kernel(const float* __restrict__ rq, const float* __restrict__ vq,
                                                          long long nchunks, float w0, float inv_cells,
                                                          float* __restrict__ out) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nchunks;
       g += (long long)gridDim.x * blockDim.x) {
    const float4* pr = reinterpret_cast<const float4*>(rq + g * QC);
    const float4* pv = reinterpret_cast<const float4*>(vq + g * QC);
    float o[QC];
    triple_chunk([&](int u) { return __ldg(pr + u); }, [&](int u) { return __ldg(pv + u); }, w0, inv_cells, o);
    float4* po = reinterpret_cast<float4*>(out + g * QC);
#pragma unroll
    for (int u = 0; u < QC / 4; ++u) po[u] = make_float4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
  }
}

// fp16 hi / lo pieces of o 2^e into the TMEM A stage at taddr.  Always scaled (sc = 1 when e = 0):
// one code path measured 4% faster than branching on rx.scaled around an unscaled copy -- the
// converter is issue-bound and the branch cost the loads' interleaving with the splits.
__device__ __forceinline__ void split_store(const float* o, float sc, uint32_t taddr) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) split_pair_scaled(o[32 * h + 2 * c], o[32 * h + 2 * c + 1], sc, hi[c], lo[c]);
    tmem_st16(taddr + h * 16, hi);
    tmem_st16(taddr + 32 + h * 16, lo);
  }
}
// ------------------------------------------------------------------------------- tensor-core kernel
constexpr int BM = 128, BK = 64, BN = 64;
constexpr int DSTAGES = 3;                      // rho + V tiles
constexpr int LSTAGES = 2;                      // light tiles
constexpr int ASTAGES = 4;                      // TMEM A stages
constexpr int KG = 16;                          // k blocks per accumulation group (relight_tc.cu)
constexpr int T_TILE = BM * BK * 4;             // 32 KB per operand tile
constexpr int D_STAGE = 2 * T_TILE;             // rho | V
constexpr int L_STAGE = kTcLTileBytes;          // 16 KB
constexpr int SMEM_TILES = DSTAGES * D_STAGE + LSTAGES * L_STAGE;
constexpr int EXP_OFF = SMEM_TILES + 256;       // int8 exponent ring [kExpRing][BM] after the barriers
constexpr int SMEM_BYTES = EXP_OFF + kExpRing * BM + 1024;
constexpr int kThreads = 384;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACC_COL0 = ASTAGES * 64;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

__global__ void __launch_bounds__(kThreads, 1)
    relight_triple_tc_kernel(const __grid_constant__ CUtensorMap tmapR, const __grid_constant__ CUtensorMap tmapV,
                             const uint8_t* __restrict__ ltiles, const float* __restrict__ inv_scale_g,
                             float* __restrict__ R, long long V, int K, int B, int ntiles, float w0, float inv_cells,
                             RedoList* __restrict__ redo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sD = smem;                                   // DSTAGES x (rho 32 KB | V 32 KB)
  uint8_t* sL = smem + DSTAGES * D_STAGE;               // LSTAGES x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_TILES);
  uint64_t* dfull = bars;                               // [DSTAGES] TMA -> converters
  uint64_t* dempty = dfull + DSTAGES;                   // [DSTAGES] converters (128) -> TMA
  uint64_t* lfull = dempty + DSTAGES;                   // [LSTAGES] bulk copy -> MMA
  uint64_t* lempty = lfull + LSTAGES;                   // [LSTAGES] MMA commit -> bulk copy
  uint64_t* afull = lempty + LSTAGES;                   // [ASTAGES] converters -> MMA
  uint64_t* aempty = afull + ASTAGES;                   // [ASTAGES] MMA commit -> converters
  uint64_t* tfull = aempty + ASTAGES;                   // [2] MMA -> epilogue
  uint64_t* tempty = tfull + 2;                         // [2] epilogue (128) -> MMA
  uint64_t* efull = tempty + 2;                         // [kExpRing] converters (128) -> epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(efull + kExpRing);
  int8_t* sexp = reinterpret_cast<int8_t*>(smem + EXP_OFF);
  static_assert((2 * DSTAGES + 2 * LSTAGES + 2 * ASTAGES + 4 + kExpRing) * 8 + 4 <= 256, "barrier block");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = K / BK;
  const int nfb = B / BN;
  const long long nwork = (long long)ntiles * nfb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < DSTAGES; ++s) {
      mbar_init(&dfull[s], 1);
      mbar_init(&dempty[s], 128);
    }
    for (int s = 0; s < LSTAGES; ++s) {
      mbar_init(&lfull[s], 1);
      mbar_init(&lempty[s], 1);
    }
    for (int s = 0; s < ASTAGES; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    for (int s = 0; s < kExpRing; ++s) mbar_init(&efull[s], 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (rho, V)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmapR) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmapV) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (long long w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int tile = (int)(w / nfb);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&dempty[stage], phase ^ 1);
          mbar_expect_tx(&dfull[stage], D_STAGE);
          uint8_t* d = sD + stage * D_STAGE;
          tma_load_2d(d, &tmapR, kb * BK, tile * BM, &dfull[stage]);
          tma_load_2d(d + T_TILE / 2, &tmapR, kb * BK + 32, tile * BM, &dfull[stage]);
          tma_load_2d(d + T_TILE, &tmapV, kb * BK, tile * BM, &dfull[stage]);
          tma_load_2d(d + T_TILE + T_TILE / 2, &tmapV, kb * BK + 32, tile * BM, &dfull[stage]);
          if (++stage == DSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------------ light tiles
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int fb = (int)(w % nfb);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&lempty[stage], phase ^ 1);
          mbar_expect_tx(&lfull[stage], L_STAGE);
          bulk_load(sL + stage * L_STAGE, ltiles + ((long long)fb * nkb + kb) * L_STAGE, L_STAGE, &lfull[stage]);
          if (++stage == LSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int lstage = 0, astage = 0;
      uint32_t lphase = 0, aphase = 0;
      int gi = 0;   // accumulation group counter: buffer gi & 1
      const uint32_t id128 = idesc_f16(2 * BN), id64 = idesc_f16(BN);
      for (long long w = blockIdx.x; w < nwork; w += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          const int acc = gi & 1;
          const bool first = (kb % KG) == 0;
          if (first) {
            mbar_wait(&tempty[acc], ((gi >> 1) & 1) ^ 1);   // the epilogue drained this buffer
            fence_after();
          }
          const uint32_t dhh = tmem + ACC_COL0 + acc * 128;
          mbar_wait(&lfull[lstage], lphase);
          mbar_wait(&afull[astage], aphase);
          fence_after();
          const uint32_t lbase = smem_u32(sL + lstage * L_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t bd = sw128_desc(lbase + kk * 32);
            const uint32_t ahi = tmem + astage * 64 + kk * 8;
            tc_mma_ts(dhh, ahi, bd, id128, (!first || kk) ? 1u : 0u);   // [acc_hh | acc_x] (=|+=) M_hi x [L_hi | L_lo]
            tc_mma_ts(dhh + BN, ahi + 32, bd, id64, 1u);                  // acc_x += M_lo x L_hi
          }
          tc_commit(&lempty[lstage]);
          tc_commit(&aempty[astage]);
          if (++lstage == LSTAGES) {
            lstage = 0;
            lphase ^= 1;
          }
          if (++astage == ASTAGES) {
            astage = 0;
            aphase ^= 1;
          }
          if ((kb % KG) == KG - 1 || kb == nkb - 1) {
            tc_commit(&tfull[acc]);
            ++gi;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------------ converters
    const int row = threadIdx.x - 128;
    const int q = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int sw = row & 7;
    int stage = 0, astage = 0;
    uint32_t phase = 0, aphase = 0;
    int tc = 0;   // tiles converted by this CTA: exponent ring slot tc & 7
    RowExp rx;
    for (long long w = blockIdx.x; w < nwork; w += gridDim.x, ++tc) {
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&dfull[stage], phase);
        mbar_wait(&aempty[astage], aphase ^ 1);
        fence_after();
        const uint8_t* tr = sD + stage * D_STAGE + row * 128;
        const uint8_t* tv = tr + T_TILE;
        float o[QC];
        triple_chunk(
            [&](int u) { return *reinterpret_cast<const float4*>(tr + (u >> 3) * (T_TILE / 2) + (((u & 7) ^ sw) << 4)); },
            [&](int u) { return *reinterpret_cast<const float4*>(tv + (u >> 3) * (T_TILE / 2) + (((u & 7) ^ sw) << 4)); },
            w0, inv_cells, o);
        rx.update(kb, [&] {
          float mx = 0.f;
#pragma unroll
          for (int i = 0; i < QC; ++i) mx = fmaxf(mx, fabsf(o[i]));
          return mx;
        });
        split_store(o, pow2i(rx.e), lane_base + astage * 64);
        if (kb == nkb - 1) {
          sexp[(tc & (kExpRing - 1)) * BM + row] = (int8_t)rx.e;
          mbar_arrive(&efull[tc & (kExpRing - 1)]);
        }
        tmem_wait_st();
        fence_before();
        mbar_arrive(&afull[astage]);
        mbar_arrive(&dempty[stage]);
        if (++stage == DSTAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++astage == ASTAGES) {
          astage = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------------ epilogue
    const int row = threadIdx.x - 256;
    const int q = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    int gi = 0, tc = 0;
    for (long long w = blockIdx.x; w < nwork; w += gridDim.x, ++tc) {
      const int tile = (int)(w / nfb), fb = (int)(w % nfb);
      const long long grow = (long long)tile * BM + row;
      float sum[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) sum[j] = 0.f;
      for (int g0 = 0; g0 < nkb; g0 += KG, ++gi) {
        const int acc = gi & 1;
        mbar_wait(&tfull[acc], (gi >> 1) & 1);
        fence_after();
#pragma unroll
        for (int c = 0; c < BN / 16; ++c) {
          float hh[16], xx[16];
          tmem_ld16(lane_base + ACC_COL0 + acc * 128 + c * 16, hh);
          tmem_ld16(lane_base + ACC_COL0 + acc * 128 + BN + c * 16, xx);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) sum[c * 16 + j] += fmaf(xx[j], 1.f / 2048.f, hh[j]);
        }
        fence_before();
        mbar_arrive(&tempty[acc]);
      }
      const int slot = tc & (kExpRing - 1);
      mbar_wait(&efull[slot], (tc / kExpRing) & 1);
      const float rs = pow2i(-(int)sexp[slot * BM + row]);   // 2^-e of this row
      if (grow < V) {
        float* out = R + grow * B + fb * BN;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < BN; j += 4) {
          float4 o;
          o.x = sum[j + 0] * rs * __ldg(inv_scale_g + fb * BN + j + 0);
          o.y = sum[j + 1] * rs * __ldg(inv_scale_g + fb * BN + j + 1);
          o.z = sum[j + 2] * rs * __ldg(inv_scale_g + fb * BN + j + 2);
          o.w = sum[j + 3] * rs * __ldg(inv_scale_g + fb * BN + j + 3);
          bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
          *reinterpret_cast<float4*>(out + j) = o;
        }
        if (bad) redo_push(redo, grow);
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

constexpr long long kFallbackRows = 16384;   // rows per materialised chunk of the CUDA-core path

int log2_of(long long x) {
  int k = 0;
  while ((1ll << k) < x) ++k;
  return k;
}

bool triple_tc_eligible(int faces, int kface, int batch) { return relight_tc_eligible(faces, kface, batch); }

struct TripleRow {   // the tripling terms of a row, chunk by chunk (relight_redo_rows_kernel)
  const float* rq;
  const float* vq;
  long long K;
  float w0, inv_cells;
  __device__ void operator()(long long row, int k0, int nk, float* sx) const {
    for (int c = threadIdx.x; c < nk / QC; c += blockDim.x) {
      const float4* pr = reinterpret_cast<const float4*>(rq + row * K + k0 + (long long)c * QC);
      const float4* pv = reinterpret_cast<const float4*>(vq + row * K + k0 + (long long)c * QC);
      triple_chunk([&](int u) { return __ldg(pr + u); }, [&](int u) { return __ldg(pv + u); }, w0, inv_cells,
                   sx + c * QC);
    }
  }
};

}  // namespace

hs_status launch_pack_qtree(const float* in, long long rows, int faces, long long in_face_stride, int log2k,
                            float* out, cudaStream_t st) {
  const long long rf = rows * faces;
  if (rf <= 0) return HS_OK;
  const unsigned gy = (unsigned)(rf < 65535 ? rf : 65535);
  const unsigned gz = (unsigned)((rf + gy - 1) / gy);
  if ((long long)gy * gz != rf) {   // ragged: launch the full 65535-row slabs, then the rest
    const long long full = (rf / gy) * gy;
    pack_qtree_kernel<<<dim3((unsigned)((1 << (2 * log2k)) + 255) / 256, gy, (unsigned)(rf / gy)), 256, 0, st>>>(
        in, faces, in_face_stride, log2k, out);
    HS_CHECK_LAUNCH("pack_qtree_kernel");
    return launch_pack_qtree(in + full * in_face_stride, rf - full, 1, in_face_stride, log2k,
                             out + (full << (2 * log2k)), st);
  }
  pack_qtree_kernel<<<dim3((unsigned)((1 << (2 * log2k)) + 255) / 256, gy, gz), 256, 0, st>>>(in, faces, in_face_stride,
                                                                                           log2k, out);
  HS_CHECK_LAUNCH("pack_qtree_kernel");
  return HS_OK;
}

// Workspace: Lq [batch][faces*kface] fp32 | tensor-core light tiles (or the fallback M chunk).
size_t relight_triple_workspace_bytes_impl(long long V, int faces, int kface, int batch) {
  const size_t lq = ((size_t)batch * faces * kface * sizeof(float) + 1023) & ~size_t(1023);
  if (triple_tc_eligible(faces, kface, batch)) return lq + relight_tc_workspace_bytes(faces, kface, batch);
  const long long rows = V < kFallbackRows ? V : kFallbackRows;
  return lq + (size_t)rows * faces * kface * sizeof(float);
}

hs_status launch_relight_triple(const float* brdf_q, const float* vis_q, long long V, int faces, int kface,
                                const float* light, long long lstride, int batch, float* R, void* ws, size_t ws_bytes,
                                cudaStream_t st) {
  const int k = log2_of(kface) / 2;
  const int r = k - 3;
  const float w0 = ldexpf(1.f, r), inv_cells = ldexpf(1.f, -2 * r);
  float* lq = reinterpret_cast<float*>(ws);
  const size_t lq_bytes = ((size_t)batch * faces * kface * sizeof(float) + 1023) & ~size_t(1023);
  uint8_t* rest = reinterpret_cast<uint8_t*>(ws) + lq_bytes;
  hs_status s = launch_pack_qtree(light, batch, faces, lstride, k, lq, st);
  if (s != HS_OK) return s;
  const long long K = (long long)faces * kface;

  if (triple_tc_eligible(faces, kface, batch)) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = get_encode();
    if (!encode) {
      set_cuda_error(cudaErrorNotSupported, "cuTensorMapEncodeTiled unavailable");
      return HS_ERR_CUDA;
    }
    s = launch_relight_tc_prep(lq, kface, faces, kface, batch, rest, st);
    if (s != HS_OK) return s;
    const float* inv = reinterpret_cast<const float*>(rest + (size_t)(batch / BN) * (size_t)(K / BK) * L_STAGE);
    CUtensorMap maps[2];
    const float* srcs[2] = {brdf_q, vis_q};
    for (int i = 0; i < 2; ++i) {
      const cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)V};
      const cuuint64_t gstride[1] = {(cuuint64_t)K * 4};
      const cuuint32_t box[2] = {32, BM};
      const cuuint32_t estr[2] = {1, 1};
      CUresult cr = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(srcs[i]), gdim, gstride,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) {
        set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled(rho/V)");
        return HS_ERR_CUDA;
      }
    }
    HS_SMEM_ATTR(relight_triple_tc_kernel, SMEM_BYTES);
    const int ntiles = (int)((V + BM - 1) / BM);
    const long long nwork = (long long)ntiles * (batch / BN);
    const int grid = (int)(nwork < num_sms() ? nwork : num_sms());
    RedoList* redo = reinterpret_cast<RedoList*>(rest + tc_redo_offset(faces, kface, batch));
    relight_triple_tc_kernel<<<grid, kThreads, SMEM_BYTES, st>>>(maps[0], maps[1], rest, inv, R, V, (int)K, batch,
                                                                 ntiles, w0, inv_cells, redo);
    HS_CHECK_LAUNCH("relight_triple_tc_kernel");
    relight_redo_rows_kernel<TripleRow><<<num_sms(), 128, 0, st>>>(TripleRow{brdf_q, vis_q, K, w0, inv_cells}, lq, K,
                                                                  kface, k * 2, (int)K, batch, R, V, redo);
    HS_CHECK_LAUNCH("relight_redo_rows_kernel");
    return HS_OK;
  }

  // CUDA-core path: materialise M for a chunk of rows, then the plain relight against Lq.
  float* m = reinterpret_cast<float*>(rest);
  for (long long r0 = 0; r0 < V; r0 += kFallbackRows) {
    const long long rows = (V - r0) < kFallbackRows ? (V - r0) : kFallbackRows;
    const long long nchunks = rows * K / QC;
    long long blocks = (nchunks + 127) / 128;
    if (blocks > (long long)num_sms() * 8) blocks = (long long)num_sms() * 8;
    triple_text_kernel<<<(unsigned)blocks, 128, 0, st>>>(brdf_q + r0 * K, vis_q + r0 * K, nchunks, w0, inv_cells, m);
    HS_CHECK_LAUNCH("triple_text_kernel");
    s = launch_relight(m, rows, faces, kface, lq, kface, batch, R + r0 * batch, nullptr, 0, st);
    if (s != HS_OK) return s;
  }
  return HS_OK;
}

}  // namespace hs
