// Internal declarations shared by the translation units of libhaarshift.so.
// Nothing here is visible through the C ABI (include/haarshift.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "haarshift.h"

namespace hs {

// ----------------------------------------------------------------------------------- errors

void set_cuda_error(cudaError_t e, const char* where);
hs_status check_device();                 // HS_ERR_UNSUPPORTED unless the current device is sm_100
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern thread_local int g_launches;       // kernel launches enqueued by the current ABI call

// Per-device state (a process may drive several GPUs): the SM count of the current device, and
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applied once per (device, kernel).
int device_sm_count();
cudaError_t ensure_max_smem(const void* kernel, int bytes);
#define HS_SMEM_ATTR(kernel, bytes) \
  HS_CHECK_CUDA(::hs::ensure_max_smem(reinterpret_cast<const void*>(kernel), (int)(bytes)), "cudaFuncSetAttribute(" #kernel ")")

#define HS_CHECK_LAUNCH(where)                                   \
  do {                                                           \
    cudaError_t e_ = cudaGetLastError();                         \
    if (e_ != cudaSuccess) {                                     \
      ::hs::set_cuda_error(e_, where);                           \
      return HS_ERR_CUDA;                                        \
    }                                                            \
    ++::hs::g_launches;                                          \
  } while (0)

#define HS_CHECK_CUDA(call, where)                               \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) {                                     \
      ::hs::set_cuda_error(e_, where);                           \
      return HS_ERR_CUDA;                                        \
    }                                                            \
  } while (0)

// ----------------------------------------------------------------------------------- shift

// Per-face shift parameters, computed in fp64 on the host (or by shift_params_kernel on the
// device for per-vertex shifts) -- SURVEY.md §8(a) row a0.
struct FaceParam {
  int m;         // working level: levels >= m are exact permutations, the recursion runs to m
  int Qy, Qx;    // integer part of the shift at level m (in level-m cells), in [0, 2^m)
  int qy, qx;    // integer part of the shift at the finest level n, in [0, N)
  float wy, wx;  // fractional parts phi (box-projection weights w1 = phi, w0 = 1 - phi)
};

// fp64 reduction s -> (q, phi): s mod N, q = floor, phi = s - q  (R4/R5).
__host__ __device__ inline void split_shift(double s, int N, int* q, double* phi) {
  double r = fmod(s, (double)N);
  if (r < 0.0) r += (double)N;
  double fq = floor(r);
  double p = r - fq;
  int qi = (int)fq;
  if (qi >= N) qi -= N;
  *q = qi;
  *phi = p;
}

__host__ __device__ inline int v2_capped(int q, int n) {  // 2-adic valuation, v2(0) = n
  if (q == 0) return n;
  int v = 0;
  while (((q >> v) & 1) == 0 && v < n) ++v;
  return v;
}

__host__ __device__ inline FaceParam make_face_param_2d(double sy, double sx, int n) {
  const int N = 1 << n;
  int qy, qx;
  double py, px;
  split_shift(sy, N, &qy, &py);
  split_shift(sx, N, &qx, &px);
  FaceParam fp;
  if (py == 0.0 && px == 0.0) {
    int v = v2_capped(qy, n);
    int vx = v2_capped(qx, n);
    if (vx < v) v = vx;
    fp.m = n - v;
  } else {
    fp.m = n;
  }
  fp.Qy = qy >> (n - fp.m);
  fp.Qx = qx >> (n - fp.m);
  fp.qy = qy;
  fp.qx = qx;
  fp.wy = (float)py;
  fp.wx = (float)px;
  return fp;
}

__host__ __device__ inline FaceParam make_face_param_1d(double s, int n) {
  const int N = 1 << n;
  int q;
  double p;
  split_shift(s, N, &q, &p);
  FaceParam fp;
  fp.m = (p == 0.0) ? n - v2_capped(q, n) : n;
  fp.Qy = 0;
  fp.Qx = q >> (n - fp.m);
  fp.qy = 0;
  fp.qx = q;
  fp.wy = 0.f;
  fp.wx = (float)p;
  return fp;
}

constexpr int kMaxFacesPerLaunch = 1024;   // ShiftArgs stays under the 32 KB kernel-parameter limit

struct ShiftArgs {
  const float* in;            // face g reads in + (g / faces) * in_batch_stride + (g % faces) * K
  float* out;                 // face g writes out + g * out_face_stride
  float* ws;                  // per-face coarse fields (see shift_workspace_layout)
  const FaceParam* dev_fp;    // device FaceParams (per-vertex path) or nullptr -> use fp[]
  long long in_batch_stride;  // elements; 0 broadcasts one pyramid set to every batch entry
  long long in_face_stride;   // elements between the faces of one batch entry (>= K)
  long long ws_face_stride;   // BYTES per face in ws (ws_face_floats_2d doubles)
  int log2n, faces, band, out_face_stride, num_faces;
  int band_path;              // 1: faces with kBandMinLevel <= m <= kBandMaxLevel go to shift2d_band_kernel
  FaceParam fp[kMaxFacesPerLaunch];
};

// Working levels handled by the band kernel (shift2d_band.cu); max_m: the largest such level present.
constexpr int kBandMinLevel = 6;
constexpr int kBandMaxLevel = 9;
inline __host__ __device__ bool band_level(int m) { return m >= kBandMinLevel && m <= kBandMaxLevel; }
hs_status launch_shift2d_band(ShiftArgs& a, int max_m, cudaStream_t st);   // shift2d_band.cu

// Tiling constants of the 2D tile kernel.
constexpr int kTileKF = 3;    // fine levels per tile: the tile root level is c = max(0, m - KF)
constexpr int kTileTC = 8;    // tile side at level c (cells)

inline int coarse_level(int m) { return m > kTileKF ? m - kTileKF : 0; }
inline long long ws_face_floats_2d(int n) {  // 8-byte elements per face
  // [shifted level-c fields 3*4^c (tile field type)][unshifted level-c fields 3*4^c (fp64)]
  // [scratch 3*4^(c-1)]
  int c = coarse_level(n);
  if (c == 0) return 0;
  return 6ll * (1ll << (2 * c)) + 3ll * (1ll << (2 * (c - 1)));
}
size_t shift_workspace_bytes_impl(int ndim, int log2n, long long num_faces);
hs_status launch_shift(const float* in, float* out, int ndim, int log2n, int faces,
                       long long num_faces, long long in_batch_stride, long long in_face_stride,
                       const double* shifts_host,
                       const float* shifts_dev_per_vertex, FaceParam* dev_fp_buf, int band,
                       void* ws, size_t ws_bytes, cudaStream_t st);

// ----------------------------------------------------------------------------------- relight

hs_status launch_relight(const float* T, long long V, int faces, int kface, const float* L,
                         long long lstride, int batch, float* R, void* ws, size_t ws_bytes, cudaStream_t st);
size_t relight_tc_workspace_bytes(int faces, int kface, int batch);
// Split-precision light tiles of the tensor-core relight (relight_tc.cu): for frame block fb (64
// frames) and k block kb (64 columns) a 16 KB pre-swizzled [L_hi | L_lo] tile at
// ws + (fb * K/64 + kb) * 16 KB, then the per-frame inverse scales (fp32 [batch]).
constexpr int kTcLTileBytes = 16384;
hs_status launch_relight_tc_prep(const float* L, long long lstride, int faces, int kface, int batch, void* ws,
                                 cudaStream_t st);
bool relight_tc_eligible(int faces, int kface, int batch);
size_t tc_redo_offset(int faces, int kface, int batch);   // RedoList (tc_ptx.cuh) inside the tc workspace
hs_status launch_rowdot(const float* T, const float* S, long long rows, long long K, float* R,
                        cudaStream_t st);
bool relight_shifted_fused_supported(int log2n);
size_t relight_shifted_fused_workspace_bytes(long long V, int faces, int log2n);
size_t relight_planes_workspace_bytes(long long V, int faces);
size_t relight_small_planes_workspace_bytes(long long V, int faces, int log2n);
hs_status launch_relight_small_planes(const float* T, long long V, int faces, const float* light, int log2n,
                                      const double* fields64, long long face_stride, const int4* vparams, float* R,
                                      void* ws, cudaStream_t st);
hs_status launch_relight_planes(const float* T, long long V, int faces, const float* light, const double* fields64,
                                long long face_stride, const int4* vparams, float* R, void* ws, cudaStream_t st);
hs_status launch_relight_shifted_fused(const float* T, long long V, int faces, const float* light, int log2n,
                                       const float* shifts, float* R, void* ws, cudaStream_t st);
hs_status launch_fill_sparse(int* idx, float* val, long long row_start, long long rows, int faces, int n, int ks,
                             int dense_levels, uint64_t seed, cudaStream_t st);
hs_status launch_relight_sparse(const int* idx, const float* val, long long V, int ks, const float* light, long long C,
                                int B, float* R, float* Lt, cudaStream_t st);
hs_status launch_pack_qtree(const float* in, long long rows, int faces, long long in_face_stride, int log2k,
                            float* out, cudaStream_t st);
size_t relight_triple_workspace_bytes_impl(long long V, int faces, int kface, int batch);
hs_status launch_relight_triple(const float* brdf_q, const float* vis_q, long long V, int faces, int kface,
                                const float* light, long long lstride, int batch, float* R, void* ws, size_t ws_bytes,
                                cudaStream_t st);
size_t rotate_workspace_bytes_impl(int log2n, long long maps);
hs_status launch_rotate(const float* in, float* out, int n, long long maps, const double* angles, void* ws,
                        size_t ws_bytes, cudaStream_t st, bool bcast = false);   // bcast: one source pyramid for all maps
size_t brdf_rotated_workspace_bytes_impl(int log2n, int log2k, int batch);
hs_status launch_relight_brdf_rotated(const float* brdf, int log2n, const double* normals, long long V, const float* vis_q,
                                      int log2k, const float* light, long long lstride, int batch, float* R, void* ws,
                                      size_t ws_bytes, cudaStream_t st);
hs_status launch_fill_transfer(float* out, long long row_start, long long rows, int faces,
                               int kface, uint64_t seed, uint64_t stream_id, cudaStream_t st);

}  // namespace hs
