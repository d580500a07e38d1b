// The paper's shading composed (SURVEY.md §8(f) f1 + f3): per
// vertex, the BRDF -- one lat-long map in the local frame of the surface, pole = normal -- is
// rotated into the global frame by the vertex normal's elevation and azimuth (theta_N, phi_N),
// directly on its Haar coefficients (row f1, rotate.cu: the chain rule on the difference fields,
// then the exact shift along phi), and the triple product of the light, the rotated BRDF and the
// vertex's visibility is taken in the Haar domain (row f3, relight_triple.cu):
//   R[v][b] = integral of  L_b * Rot(theta_v, phi_v) rho * V_v      (band-limited to 4^k coefficients)
// Chunks of kChunk vertices: rotate (one source pyramid for the whole chunk: its fields and pole
// rows are built once), pack the rotated bands to the qtree layout, triple-product relight of the
// chunk's rows.  Every step is one of the library's kernels; nothing goes through the host.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hs {
namespace {
constexpr long long kChunk = 4096;   // vertices per rotation batch (4 launch sequences of 1024 maps)

size_t al1k(size_t b) { return (b + 1023) & ~size_t(1023); }   // 1 KB: the triple workspace's alignment
}  // namespace

size_t brdf_rotated_workspace_bytes_impl(int log2n, int log2k, int batch) {
  const size_t NN = (size_t)1 << (2 * log2n), kf = (size_t)1 << (2 * log2k);
  return al1k(kChunk * NN * 4) + al1k(kChunk * kf * 4) + al1k(rotate_workspace_bytes_impl(log2n, kChunk)) +
         al1k(relight_triple_workspace_bytes_impl(kChunk, 1, (int)kf, batch));
}

hs_status launch_relight_brdf_rotated(const float* brdf, int log2n, const double* normals, long long V, const float* vis_q,
                                      int log2k, const float* light, long long lstride, int batch, float* R, void* ws,
                                      size_t ws_bytes, cudaStream_t st) {
  const size_t NN = (size_t)1 << (2 * log2n), kf = (size_t)1 << (2 * log2k);
  char* base = reinterpret_cast<char*>(ws);
  float* rot = reinterpret_cast<float*>(base);
  float* qt = reinterpret_cast<float*>(base + al1k(kChunk * NN * 4));
  void* rws = base + al1k(kChunk * NN * 4) + al1k(kChunk * kf * 4);
  const size_t rws_bytes = al1k(rotate_workspace_bytes_impl(log2n, kChunk));
  void* tws = reinterpret_cast<char*>(rws) + rws_bytes;
  const size_t tws_bytes = ws_bytes - (al1k(kChunk * NN * 4) + al1k(kChunk * kf * 4) + rws_bytes);
  for (long long v0 = 0; v0 < V; v0 += kChunk) {
    const long long cv = (V - v0) < kChunk ? (V - v0) : kChunk;
    // (alpha, beta) = (theta_N, phi_N): elevation then azimuth (R28)
    hs_status s = launch_rotate(brdf, rot, log2n, cv, normals + 2 * v0, rws, rws_bytes, st, /*bcast=*/true);
    if (s != HS_OK) return s;
    s = launch_pack_qtree(rot, cv, 1, (long long)NN, log2k, qt, st);
    if (s != HS_OK) return s;
    s = launch_relight_triple(qt, vis_q + v0 * (long long)kf, cv, 1, (int)kf, light, lstride, batch, R + v0 * batch,
                              tws, tws_bytes, st);
    if (s != HS_OK) return s;
  }
  return HS_OK;
}

}  // namespace hs
