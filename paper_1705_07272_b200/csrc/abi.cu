// C-ABI entry points (include/haarshift.h): argument validation before any launch, status codes,
// thread-local error detail.  No CPU fallback, no other backend.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace hs {

thread_local int g_launches = 0;
namespace {
thread_local char g_err[512] = "";
thread_local int g_last_launches = 0;
std::atomic<int> g_dev_ok[64];  // 0 unknown, 1 sm_100, 2 other

inline bool is_pow4(long long x) {
  if (x < 1 || (x & (x - 1))) return false;
  int b = 0;
  while ((1ll << b) < x) ++b;
  return (b & 1) == 0;
}
inline bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}
inline bool aligned_to(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
// bytes spanned by `rows` rows of `row_len` floats at a row stride of `stride` floats
inline size_t span_bytes(long long rows, long long stride, long long row_len) {
  return (size_t)((rows - 1) * stride + row_len) * sizeof(float);
}
constexpr long long kRelightChunk = 128;  // vertices per chunk of the per-vertex shift path

}  // namespace

void set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

int device_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

cudaError_t ensure_max_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::tuple<int, const void*, int>> done;   // (device, kernel, bytes) already set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (std::get<0>(d) == dev && std::get<1>(d) == kernel && std::get<2>(d) >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(dev, kernel, bytes);
  return e;
}

hs_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_cuda_error(e, "cudaGetDevice");
    return HS_ERR_CUDA;
  }
  if (dev < 0 || dev >= 64) return HS_ERR_UNSUPPORTED;
  int st = g_dev_ok[dev].load(std::memory_order_relaxed);
  if (st == 0) {
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) {
      set_cuda_error(e, "cudaDeviceGetAttribute");
      return HS_ERR_CUDA;
    }
    st = (major == 10 && minor == 0) ? 1 : 2;
    g_dev_ok[dev].store(st, std::memory_order_relaxed);
  }
  if (st != 1) {
    snprintf(g_err, sizeof(g_err), "device %d is not sm_100 (B200); this library is sm_100a only", dev);
    return HS_ERR_UNSUPPORTED;
  }
  return HS_OK;
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_abi_version(void) { return 1; }

const char* hs_status_string(hs_status s) {
  switch (s) {
    case HS_OK: return "HS_OK";
    case HS_ERR_INVALID_ARG: return "HS_ERR_INVALID_ARG";
    case HS_ERR_ALIGNMENT: return "HS_ERR_ALIGNMENT";
    case HS_ERR_UNSUPPORTED: return "HS_ERR_UNSUPPORTED";
    case HS_ERR_CUDA: return "HS_ERR_CUDA";
  }
  return "HS_ERR_UNKNOWN";
}

const char* hs_last_cuda_error(void) { return g_err; }
int hs_last_launch_count(void) { return g_last_launches; }

size_t haar_shift_workspace_bytes(int ndim, int log2n, int faces, int batch) {
  if ((ndim != 1 && ndim != 2) || log2n < 1 || log2n > HS_MAX_LOG2N || faces < 1 || batch < 1) return 0;
  return shift_workspace_bytes_impl(ndim, log2n, (long long)faces * batch);
}

hs_status haar_shift_coeffs(const float* in, float* out, int ndim, int log2n, int faces, int batch,
                            const double* shifts_host, int band_levels, void* workspace,
                            size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!in || !out || !shifts_host) return HS_ERR_INVALID_ARG;
  if (ndim != 1 && ndim != 2) return HS_ERR_INVALID_ARG;
  if (log2n < 1 || log2n > HS_MAX_LOG2N || faces < 1 || faces > HS_MAX_FACES || batch < 1) return HS_ERR_INVALID_ARG;
  if (band_levels < 0 || band_levels > log2n) return HS_ERR_INVALID_ARG;
  const long long nfaces = (long long)faces * batch;
  for (long long i = 0; i < nfaces * ndim; ++i)
    if (!std::isfinite(shifts_host[i])) return HS_ERR_INVALID_ARG;
  const size_t K = (ndim == 2) ? ((size_t)1 << (2 * log2n)) : ((size_t)1 << log2n);
  const size_t Kb = (ndim == 2) ? ((size_t)1 << (2 * band_levels)) : ((size_t)1 << band_levels);
  if (overlap(in, nfaces * K * 4, out, nfaces * Kb * 4)) return HS_ERR_INVALID_ARG;
  const size_t need = shift_workspace_bytes_impl(ndim, log2n, nfaces);
  if (need > 0 && (!workspace || workspace_bytes < need)) return HS_ERR_INVALID_ARG;
  if (!aligned16(in) || !aligned16(out) || (need > 0 && !aligned16(workspace))) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_shift(in, out, ndim, log2n, faces, nfaces, (long long)faces * (long long)K, (long long)K, shifts_host,
                   nullptr, nullptr, band_levels, workspace, workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

size_t haar_shift_coarse_workspace_bytes(int in_log2n, int start_level, int faces, int batch) {
  if (in_log2n < 1 || in_log2n > HS_MAX_LOG2N || start_level < 1 || start_level > in_log2n) return 0;
  return haar_shift_workspace_bytes(2, start_level, faces, batch);
}

hs_status haar_shift_coeffs_coarse(const float* in, float* out, int in_log2n, int start_level, int faces, int batch,
                                   const double* shifts_host, int band_levels, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!in || !out || !shifts_host) return HS_ERR_INVALID_ARG;
  if (in_log2n < 1 || in_log2n > HS_MAX_LOG2N || start_level < 1 || start_level > in_log2n) return HS_ERR_INVALID_ARG;
  if (faces < 1 || faces > HS_MAX_FACES || batch < 1 || band_levels < 0 || band_levels > start_level)
    return HS_ERR_INVALID_ARG;
  const long long nfaces = (long long)faces * batch;
  for (long long i = 0; i < nfaces * 2; ++i)
    if (!std::isfinite(shifts_host[i])) return HS_ERR_INVALID_ARG;
  const size_t K = (size_t)1 << (2 * in_log2n);
  const size_t Kb = (size_t)1 << (2 * band_levels);
  if (overlap(in, nfaces * K * 4, out, nfaces * Kb * 4)) return HS_ERR_INVALID_ARG;
  const size_t need = shift_workspace_bytes_impl(2, start_level, nfaces);
  if (need > 0 && (!workspace || workspace_bytes < need)) return HS_ERR_INVALID_ARG;
  if (!aligned16(in) || !aligned16(out) || (need > 0 && !aligned16(workspace))) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  // the level-L approximation is the HAAR1 prefix; a shift of s pixels moves it by s / 2^(n-L) cells
  std::vector<double> sc((size_t)nfaces * 2);
  const double inv = std::ldexp(1.0, -(in_log2n - start_level));
  for (size_t i = 0; i < sc.size(); ++i) sc[i] = shifts_host[i] * inv;
  s = launch_shift(in, out, 2, start_level, faces, nfaces, (long long)faces * (long long)K, (long long)K, sc.data(),
                   nullptr, nullptr, band_levels, workspace, workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

size_t relight_workspace_bytes(int faces, int k_face, int batch) {
  if (faces < 1 || batch < 1 || batch > 1024 || !is_pow4(k_face) || k_face < 4) return 0;
  return relight_tc_workspace_bytes(faces, k_face, batch);
}

hs_status relight_vertices(const float* transfer, int64_t num_vertices, int faces, int k_face,
                           const float* light, int64_t light_face_stride, int batch, float* radiance,
                           void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!transfer || !light || !radiance) return HS_ERR_INVALID_ARG;
  if (num_vertices < 1 || faces < 1 || batch < 1 || batch > 1024) return HS_ERR_INVALID_ARG;
  if (!is_pow4(k_face) || k_face < 4 || k_face > (1 << (2 * HS_MAX_LOG2N))) return HS_ERR_INVALID_ARG;
  if (light_face_stride < k_face || (light_face_stride & 3)) return HS_ERR_INVALID_ARG;
  if ((long long)faces * k_face > (1ll << 30)) return HS_ERR_INVALID_ARG;
  const size_t need = relight_tc_workspace_bytes(faces, k_face, batch);
  if (need > 0 && (!workspace || workspace_bytes < need)) return HS_ERR_INVALID_ARG;
  {
    const long long K = (long long)faces * k_face;
    const size_t rb = (size_t)num_vertices * batch * sizeof(float);
    if (overlap(radiance, rb, transfer, (size_t)num_vertices * K * 4) ||
        overlap(radiance, rb, light, span_bytes((long long)batch * faces, light_face_stride, k_face)) ||
        (need > 0 && overlap(radiance, rb, workspace, need)))
      return HS_ERR_INVALID_ARG;
  }
  // the tensor-core epilogue stores float4 rows; the CUDA-core paths store single floats
  if (!aligned16(transfer) || !aligned16(light) || !aligned_to(radiance, need > 0 ? 16 : 4) ||
      (need > 0 && (reinterpret_cast<uintptr_t>(workspace) & 1023)))
    return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_relight(transfer, num_vertices, faces, k_face, light, light_face_stride, batch, radiance, workspace,
                     workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

size_t relight_shifted_workspace_bytes(int64_t num_vertices, int faces, int log2n) {
  if (num_vertices < 1 || faces < 1 || log2n < 1 || log2n > HS_MAX_LOG2N) return 0;
  if (relight_shifted_fused_supported(log2n)) return relight_shifted_fused_workspace_bytes(num_vertices, faces, log2n);
  const long long vc = num_vertices < kRelightChunk ? num_vertices : kRelightChunk;
  const long long nf = vc * faces;
  const size_t shift_ws = shift_workspace_bytes_impl(2, log2n, nf);
  const size_t fp = ((size_t)nf * sizeof(FaceParam) + 255) & ~(size_t)255;
  const size_t pyr = (size_t)nf * ((size_t)1 << (2 * log2n)) * sizeof(float);
  return shift_ws + fp + pyr;
}

hs_status relight_vertices_shifted(const float* transfer, int64_t num_vertices, int faces, const float* light,
                                   int log2n, const float* vertex_shifts, float* radiance, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!transfer || !light || !vertex_shifts || !radiance || !workspace) return HS_ERR_INVALID_ARG;
  if (num_vertices < 1 || faces < 1 || faces > HS_MAX_FACES || log2n < 1 || log2n > HS_MAX_LOG2N)
    return HS_ERR_INVALID_ARG;
  {
    const long long K = (long long)faces << (2 * log2n);
    const size_t rb = (size_t)num_vertices * sizeof(float);
    if (overlap(radiance, rb, transfer, (size_t)num_vertices * K * 4) || overlap(radiance, rb, light, (size_t)K * 4) ||
        overlap(radiance, rb, vertex_shifts, (size_t)num_vertices * 8))
      return HS_ERR_INVALID_ARG;
  }
  const size_t need = relight_shifted_workspace_bytes(num_vertices, faces, log2n);
  if (workspace_bytes < need) return HS_ERR_INVALID_ARG;
  if (!aligned16(transfer) || !aligned16(light) || !aligned_to(radiance, 4) || !aligned16(workspace) ||
      (reinterpret_cast<uintptr_t>(vertex_shifts) & 7))
    return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (relight_shifted_fused_supported(log2n)) {
    s = launch_relight_shifted_fused(transfer, num_vertices, faces, light, log2n, vertex_shifts, radiance, workspace,
                                     st);
    g_last_launches = g_launches;
    return s;
  }
  const long long vc = num_vertices < kRelightChunk ? num_vertices : kRelightChunk;
  const long long K = (long long)faces << (2 * log2n);
  const size_t shift_ws = shift_workspace_bytes_impl(2, log2n, vc * faces);
  const size_t fpb = ((size_t)vc * faces * sizeof(FaceParam) + 255) & ~(size_t)255;
  char* base = (char*)workspace;
  FaceParam* fp = reinterpret_cast<FaceParam*>(base + shift_ws);
  float* S = reinterpret_cast<float*>(base + shift_ws + fpb);
  for (long long v0 = 0; v0 < num_vertices; v0 += vc) {
    const long long nv = (num_vertices - v0) < vc ? (num_vertices - v0) : vc;
    s = launch_shift(light, S, 2, log2n, faces, nv * faces, 0, 1ll << (2 * log2n), nullptr, vertex_shifts + 2 * v0,
                     fp, log2n, workspace, shift_ws, st);
    if (s != HS_OK) break;
    s = launch_rowdot(transfer + v0 * K, S, nv, K, radiance + v0, st);
    if (s != HS_OK) break;
  }
  g_last_launches = g_launches;
  return s;
}

size_t relight_sparse_workspace_bytes(int64_t total_coeffs, int batch) {
  if (total_coeffs < 1 || batch < 1 || batch > 1024) return 0;
  return (size_t)total_coeffs * (size_t)batch * sizeof(float);
}

hs_status relight_vertices_sparse(const int32_t* indices, const float* values, int64_t num_vertices, int k_sparse,
                                  const float* light, int64_t total_coeffs, int batch, float* radiance,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!indices || !values || !light || !radiance || !workspace) return HS_ERR_INVALID_ARG;
  if (num_vertices < 1 || k_sparse < 1 || total_coeffs < 1 || total_coeffs >= (1ll << 31)) return HS_ERR_INVALID_ARG;
  if (batch < 1 || batch > 1024) return HS_ERR_INVALID_ARG;
  if (workspace_bytes < relight_sparse_workspace_bytes(total_coeffs, batch)) return HS_ERR_INVALID_ARG;
  {
    const size_t rb = (size_t)num_vertices * batch * sizeof(float);
    const size_t pb = (size_t)num_vertices * k_sparse * 4;
    if (overlap(radiance, rb, indices, pb) || overlap(radiance, rb, values, pb) ||
        overlap(radiance, rb, light, (size_t)batch * total_coeffs * 4) || overlap(radiance, rb, workspace, workspace_bytes))
      return HS_ERR_INVALID_ARG;
  }
  // the 64-frame kernel stores float2 pairs; the scalar kernel single floats
  if (!aligned16(indices) || !aligned16(values) || !aligned16(light) || !aligned_to(radiance, batch >= 64 ? 8 : 4) ||
      !aligned16(workspace))
    return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_relight_sparse(indices, values, num_vertices, k_sparse, light, total_coeffs, batch, radiance,
                            reinterpret_cast<float*>(workspace), (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

hs_status hs_enable_peer_access(int peer_device) {
  g_last_launches = 0;
  g_launches = 0;
  int dev = 0, n = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    set_cuda_error(e, "cudaGetDevice");
    return HS_ERR_CUDA;
  }
  if (peer_device < 0 || peer_device >= n) return HS_ERR_INVALID_ARG;
  if (peer_device == dev) return HS_OK;
  int can = 0;
  e = cudaDeviceCanAccessPeer(&can, dev, peer_device);
  if (e != cudaSuccess) {
    set_cuda_error(e, "cudaDeviceCanAccessPeer");
    return HS_ERR_CUDA;
  }
  if (!can) {
    snprintf(g_err, sizeof(g_err), "device %d cannot access device %d", dev, peer_device);
    return HS_ERR_UNSUPPORTED;
  }
  e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return HS_OK;
  }
  if (e != cudaSuccess) {
    set_cuda_error(e, "cudaDeviceEnablePeerAccess");
    return HS_ERR_CUDA;
  }
  return HS_OK;
}

size_t haar_rotate_workspace_bytes(int log2n, int batch) {
  if (log2n < 1 || log2n > 11 || batch < 1) return 0;
  return rotate_workspace_bytes_impl(log2n, batch);
}

hs_status haar_rotate_coeffs(const float* in, float* out, int log2n, int batch, const double* angles_host,
                             void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!in || !out || !angles_host || !workspace) return HS_ERR_INVALID_ARG;
  if (log2n < 1 || log2n > 11 || batch < 1) return HS_ERR_INVALID_ARG;
  for (long long i = 0; i < 2ll * batch; ++i)
    if (!std::isfinite(angles_host[i])) return HS_ERR_INVALID_ARG;
  const size_t K = (size_t)1 << (2 * log2n);
  if (overlap(in, (size_t)batch * K * 4, out, (size_t)batch * K * 4)) return HS_ERR_INVALID_ARG;
  if (workspace_bytes < rotate_workspace_bytes_impl(log2n, batch)) return HS_ERR_INVALID_ARG;
  if (!aligned16(in) || !aligned16(out) || !aligned16(workspace)) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_rotate(in, out, log2n, batch, angles_host, workspace, workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

size_t relight_brdf_rotated_workspace_bytes(int log2n, int log2k, int batch) {
  if (log2n < 3 || log2n > 11 || log2k < 3 || log2k > log2n || batch < 1 || batch > 1024) return 0;
  return brdf_rotated_workspace_bytes_impl(log2n, log2k, batch);
}

hs_status relight_vertices_brdf_rotated(const float* brdf, int log2n, const double* normals_host, int64_t num_vertices,
                                        const float* vis_q, int log2k, const float* light, int64_t light_stride,
                                        int batch, float* radiance, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!brdf || !normals_host || !vis_q || !light || !radiance || !workspace) return HS_ERR_INVALID_ARG;
  if (log2n < 3 || log2n > 11 || log2k < 3 || log2k > log2n || num_vertices < 1 || batch < 1 || batch > 1024)
    return HS_ERR_INVALID_ARG;
  const long long kf = 1ll << (2 * log2k);
  if (light_stride < kf || (light_stride & 3)) return HS_ERR_INVALID_ARG;
  for (long long i = 0; i < 2ll * num_vertices; ++i)
    if (!std::isfinite(normals_host[i])) return HS_ERR_INVALID_ARG;
  if (workspace_bytes < brdf_rotated_workspace_bytes_impl(log2n, log2k, batch)) return HS_ERR_INVALID_ARG;
  {
    const size_t rb = (size_t)num_vertices * batch * sizeof(float);
    if (overlap(radiance, rb, brdf, ((size_t)1 << (2 * log2n)) * 4) ||
        overlap(radiance, rb, vis_q, (size_t)num_vertices * kf * 4) ||
        overlap(radiance, rb, light, span_bytes(batch, light_stride, kf)) || overlap(radiance, rb, workspace, workspace_bytes))
      return HS_ERR_INVALID_ARG;
  }
  if (!aligned16(brdf) || !aligned16(vis_q) || !aligned16(light) ||
      !aligned_to(radiance, relight_tc_eligible(1, (int)kf, batch) ? 16 : 4) ||
      (reinterpret_cast<uintptr_t>(workspace) & 1023))
    return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_relight_brdf_rotated(brdf, log2n, normals_host, num_vertices, vis_q, log2k, light, light_stride, batch,
                                  radiance, workspace, workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

hs_status haar_pack_qtree(const float* in, int64_t rows, int faces, int64_t in_face_stride, int log2k, float* out,
                          void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!in || !out || rows < 1 || faces < 1 || log2k < 3 || log2k > HS_MAX_LOG2N) return HS_ERR_INVALID_ARG;
  const long long kf = 1ll << (2 * log2k);
  if (in_face_stride < kf) return HS_ERR_INVALID_ARG;
  if (overlap(in, (size_t)((rows * faces - 1) * in_face_stride + kf) * 4, out, (size_t)(rows * faces * kf) * 4))
    return HS_ERR_INVALID_ARG;
  if (!aligned16(in) || !aligned16(out)) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_pack_qtree(in, rows, faces, in_face_stride, log2k, out, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

size_t relight_triple_workspace_bytes(int64_t num_vertices, int faces, int k_face, int batch) {
  if (num_vertices < 1 || faces < 1 || batch < 1 || batch > 1024 || !is_pow4(k_face) || k_face < 64) return 0;
  return relight_triple_workspace_bytes_impl(num_vertices, faces, k_face, batch);
}

hs_status relight_vertices_triple(const float* brdf_q, const float* vis_q, int64_t num_vertices, int faces, int k_face,
                                  const float* light, int64_t light_face_stride, int batch, float* radiance,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!brdf_q || !vis_q || !light || !radiance || !workspace) return HS_ERR_INVALID_ARG;
  if (num_vertices < 1 || faces < 1 || batch < 1 || batch > 1024) return HS_ERR_INVALID_ARG;
  if (!is_pow4(k_face) || k_face < 64 || k_face > (1 << (2 * HS_MAX_LOG2N))) return HS_ERR_INVALID_ARG;
  if (light_face_stride < k_face || (light_face_stride & 3)) return HS_ERR_INVALID_ARG;
  if ((long long)faces * k_face > (1ll << 30)) return HS_ERR_INVALID_ARG;
  if (workspace_bytes < relight_triple_workspace_bytes_impl(num_vertices, faces, k_face, batch)) return HS_ERR_INVALID_ARG;
  {
    const size_t rb = (size_t)num_vertices * batch * sizeof(float);
    const size_t qb = (size_t)num_vertices * faces * k_face * 4;
    if (overlap(radiance, rb, brdf_q, qb) || overlap(radiance, rb, vis_q, qb) ||
        overlap(radiance, rb, light, span_bytes((long long)batch * faces, light_face_stride, k_face)) ||
        overlap(radiance, rb, workspace, workspace_bytes))
      return HS_ERR_INVALID_ARG;
  }
  if (!aligned16(brdf_q) || !aligned16(vis_q) || !aligned16(light) ||
      !aligned_to(radiance, relight_tc_eligible(faces, k_face, batch) ? 16 : 4) ||
      (reinterpret_cast<uintptr_t>(workspace) & 1023))
    return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_relight_triple(brdf_q, vis_q, num_vertices, faces, k_face, light, light_face_stride, batch, radiance,
                            workspace, workspace_bytes, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

hs_status hs_fill_sparse_transfer(int32_t* indices, float* values, int64_t row_start, int64_t row_count, int faces,
                                  int log2n, int k_sparse, int dense_levels, uint64_t seed, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!indices || !values || row_start < 0 || row_count < 1 || faces < 1) return HS_ERR_INVALID_ARG;
  if (log2n < 1 || log2n > HS_MAX_LOG2N || dense_levels < 0 || dense_levels > log2n) return HS_ERR_INVALID_ARG;
  if (k_sparse < (faces << (2 * dense_levels)) || (long long)faces << (2 * log2n) >= (1ll << 31)) return HS_ERR_INVALID_ARG;
  if (k_sparse > (faces << (2 * dense_levels)) && dense_levels >= log2n) return HS_ERR_INVALID_ARG;   // no level to draw
  if (!aligned16(indices) || !aligned16(values)) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_fill_sparse(indices, values, row_start, row_count, faces, log2n, k_sparse, dense_levels, seed,
                         (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

hs_status hs_fill_transfer(float* out, int64_t row_start, int64_t row_count, int faces, int k_face,
                           uint64_t seed, uint64_t stream_id, void* stream) {
  g_last_launches = 0;
  g_launches = 0;
  if (!out || row_start < 0 || row_count < 1 || faces < 1) return HS_ERR_INVALID_ARG;
  if (!is_pow4(k_face)) return HS_ERR_INVALID_ARG;
  if (!aligned16(out)) return HS_ERR_ALIGNMENT;
  hs_status s = check_device();
  if (s != HS_OK) return s;
  s = launch_fill_transfer(out, row_start, row_count, faces, k_face, seed, stream_id, (cudaStream_t)stream);
  g_last_launches = g_launches;
  return s;
}

}  // extern "C"
