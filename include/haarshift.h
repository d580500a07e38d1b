/* haarshift.h -- C ABI of the B200-native Haar-domain shift + relight hot path.
 *
 * Method: Alnasser & Foroosh, "Non-Linear Phase-Shifting of Haar Wavelets for Run-Time
 * All-Frequency Lighting" (arXiv 1705.07272), /root/reference/PAPER.md cited as P:<line>.
 * Conventions and every reading of the paper: DESIGN.md §2, §4.
 *
 * Data conventions (all entry points)
 *   - A 2D face of side N = 2^log2n holds N*N fp32 unit-square orthonormal Haar coefficients in
 *     HAAR1 order: index 0 = scaling; level l (0 <= l < log2n), type t (H=0, V=1,
 *     D=2), cell (i, j) at 4^l*(1+t) + i*2^l + j.  Wavelet signs: H + left half,
 *     V + top half, D + main diagonal.  Rows = theta (top first), columns = phi.
 *   - A 1D signal of length N holds N fp32 unit-interval Haar coefficients: index 0 = scaling,
 *     level l cell k at 2^l + k.
 *   - Every face is an independent N x N periodic signal (cube faces are compressed separately,
 *     P:306-312; R3).
 *   - A shift s (finest-pixel units) maps f'(x) = f(x - s) followed by the box projection onto
 *     the same pixels (R4, R5): content moves to higher indices; shifts are (sy, sx).
 *
 * Memory and ownership
 *   - Unless stated otherwise pointers are CUDA DEVICE pointers owned by the caller; the library
 *     keeps no pointer after return.  Work is enqueued on `stream` (cudaStream_t passed as
 *     void*; NULL = legacy default stream) and returns without synchronising; buffers must stay
 *     valid until the stream work completes.
 *   - All device pointers must be 16-byte aligned (HS_ERR_ALIGNMENT otherwise).
 *   - Stateless and re-entrant; safe to call concurrently from several host threads on
 *     different streams with distinct workspaces.  Capturable into a CUDA graph.
 *
 * Errors
 *   - Every entry point validates all arguments BEFORE enqueuing any work and returns a status.
 *     No exceptions cross the ABI, nothing calls exit(), there is no CPU fallback and no other
 *     backend: on a device that is not sm_100 the call fails with HS_ERR_UNSUPPORTED.
 *   - HS_ERR_CUDA: a CUDA runtime error at launch; hs_last_cuda_error() returns the detail string
 *     (thread-local, valid until the next call on the same thread).
 */
#ifndef HAARSHIFT_H_
#define HAARSHIFT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HS_API __attribute__((visibility("default")))
#else
#define HS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HS_OK = 0,
  HS_ERR_INVALID_ARG = 1,  /* null pointer, size out of range, non-finite shift, in == out ... */
  HS_ERR_ALIGNMENT = 2,    /* a device pointer is not 16-byte aligned                         */
  HS_ERR_UNSUPPORTED = 3,  /* device is not sm_100 (B200), or a shape this build does not cover */
  HS_ERR_CUDA = 4          /* CUDA runtime error; see hs_last_cuda_error()                     */
} hs_status;

#define HS_MAX_LOG2N 12
#define HS_MAX_FACES 1024   /* faces per batch entry of the shift entry points (one launch's parameter block) */

/* ---------------------------------------------------------------------------------------------
 * haar_shift_coeffs -- shift of Haar coefficient pyramids computed directly in the Haar domain
 * (SURVEY.md §8(a) rows a0-a5).
 *
 * Defines:  P:459 ("a rotation with respect to the azimuth angle ... becomes a linear shift"),
 *           P:503-508 (all rotations = rotation about the theta-axis + "a simple shifting along
 *           the phi-axis"), P:331/P:408/P:463 (coefficients are finite differences), eq:pde1-2
 *           P:416-425 with identity Jacobian (the difference fields translate), eq:conv/eq:tker/
 *           eq:sker P:466-478 and P:486-497 (recursive [1,1] x [1,2,1] synthesis, O(N))
 *           (start at a coarser level: exact here for dyadic shifts).  Working levels m = 6..9
 *           (fractional shifts at N = 64..512) carry the fields' common antiderivative -- the
 *           level-m approximation of the shifted window rows, from the details only (scaling
 *           coefficient 0) -- in one fp64 field instead of three difference fields; the recursions
 *           are the same linear maps (DESIGN.md §4.1 "Band kernel").
 *
 *   in, out       [batch][faces][K] fp32, K = N*N (ndim = 2) or N (ndim = 1), HAAR1 order.
 *                 out must not overlap in.  With band_levels < log2n, out is
 *                 [batch][faces][Kb] with Kb = 4^band_levels (2D) or 2^band_levels (1D): the
 *                 HAAR1 prefix holding the scaling coefficient and levels < band_levels.
 *   ndim          1 or 2.
 *   log2n         1 .. HS_MAX_LOG2N (N = 2^log2n).
 *   faces         1 .. HS_MAX_FACES;  batch >= 1 (any count: launches are chunked by batch entry).
 *   shifts_host   HOST pointer, [batch][faces][ndim] fp64, (sy, sx) order in 2D, any finite real
 *                 value (reduced mod N internally in fp64).
 *   band_levels   0 .. log2n (log2n = full pyramid).
 *   workspace     device scratch of at least haar_shift_workspace_bytes(...) bytes (may be NULL
 *                 when that size is 0).  Contents on entry are irrelevant.
 * Result: out = S_s in, equal to forward(box_shift(inverse(in))) within fp32 output rounding:
 * the 2D fields are carried in fp64 at every size because fp32 field rounding is amplified
 * ~2^(n-l) on the coarse outputs.
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status haar_shift_coeffs(const float* in, float* out, int ndim, int log2n, int faces,
                            int batch, const double* shifts_host, int band_levels,
                            void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t haar_shift_workspace_bytes(int ndim, int log2n, int faces, int batch);

/* ---------------------------------------------------------------------------------------------
 * haar_shift_coeffs_coarse -- coarse-start shift (R23).
 *
 * Defines:  P:520 ("one can start at any resolution level that is lower than n-1. In that case,
 *           the computational complexity is reduced to O(N/4^k), where k is the number of levels
 *           removed").  Computes the shift of the level-L approximation of each face: the HAAR1
 *           prefix of levels < L (a 2^L x 2^L map of cell means) shifted by s / 2^(n-L) cells with
 *           the same exact Haar-domain method, in O(4^L).  Equal to the exact shift's levels < L
 *           when s is a multiple of 2^(n-L); an approximation of them otherwise (accuracy study:
 *           tests/test_gpu_coarse.py).
 *
 *   in            [batch][faces][4^in_log2n] fp32 HAAR1 pyramids (only the prefix is read).
 *   out           [batch][faces][4^band_levels], band_levels <= start_level.
 *   in_log2n      1 .. HS_MAX_LOG2N;  start_level L: 1 .. in_log2n.
 *   shifts_host   HOST [batch][faces][2] fp64 shifts in finest-pixel units (as haar_shift_coeffs).
 *   workspace     >= haar_shift_coarse_workspace_bytes(...).
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status haar_shift_coeffs_coarse(const float* in, float* out, int in_log2n, int start_level, int faces,
                                          int batch, const double* shifts_host, int band_levels,
                                          void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t haar_shift_coarse_workspace_bytes(int in_log2n, int start_level, int faces, int batch);

/* ---------------------------------------------------------------------------------------------
 * relight_vertices -- per-vertex light-transport inner product.
 *
 * Defines:  eq:tripleSum P:253-266 with the Tripling Coefficient Theorem's scaling case
 *           (P:287): with the transfer vector holding BRDF x visibility (PRT transfer,
 *           P:213-222) the triple sum is the coefficient dot product; "the rotated data is
 *           plugged in the triple integral computation".
 *
 *   radiance[v][b] = sum_{f < faces} sum_{k < k_face} transfer[v][f*k_face + k]
 *                                                     * light[b][f][k]   (light row stride below)
 *   transfer      [num_vertices][faces*k_face] fp32 row-major (64-bit indexing).
 *   light         [batch][faces][light_face_stride] fp32; only the first k_face entries of each
 *                 face are read, so a full shifted pyramid (stride N*N) or a band (stride k_face)
 *                 can be passed.  light_face_stride >= k_face and a multiple of 4.
 *   k_face        a power of 4 (the HAAR1 prefix 4^k: scaling + levels < k), >= 4.
 *   batch         1 .. 1024 light/rotation frames.
 *   radiance      [num_vertices][batch] fp32, must not overlap transfer, light or workspace
 *                 (HS_ERR_INVALID_ARG); 16-byte aligned when the tensor-core path runs (workspace
 *                 size > 0), 4-byte aligned otherwise (HS_ERR_ALIGNMENT).
 *   workspace     device scratch of >= relight_workspace_bytes(faces, k_face, batch) bytes,
 *                 1024-byte aligned (may be NULL when that size is 0).
 * Accumulation is fp32.  batch <= 8: CUDA-core streaming GEMV.  batch a multiple of 64 with
 * faces*k_face a multiple of 64: tcgen05 tensor-core GEMM in split-precision fp16.  Every light
 * frame is scaled by a power of two s_b and every transfer row by a power of two 2^e picked from its
 * first nonzero 64-k block (e = 0 when that block's max |T| is in [2^-4, 2^8), else the block's max
 * is moved to [2^7, 2^8)); then x = hi + 2^-11 lo in fp16 pieces, three products per 64-k block
 * accumulate in fp32 in TMEM, drained into fp32 registers every 1024 k, times 2^-e / s_b at the end.
 * Contract: ~2^-21 relative per product for every value within 2^22 binades below the row's first
 * nonzero block's max; a row with a later block more than 2^8 times larger than that (fp16
 * overflow) comes out non-finite from the tensor cores, is listed by the kernel and recomputed
 * exactly on the CUDA cores (fp64 accumulation, relight_redo_rows_kernel), so any finite fp32
 * transfer and light values give a result accurate to ~1e-6 relative per row.  Each row's
 * arithmetic depends on that row only (results are bitwise independent of row sharding).  Tested
 * at T scaled by 2^-30 ... 2^60, 1e-30, and with mixed row / block / element magnitudes
 * (tests/test_gpu_range.py).  Other batches: CUDA-core tiled
 * GEMM (fp32 FMA).
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status relight_vertices(const float* transfer, int64_t num_vertices, int faces, int k_face,
                           const float* light, int64_t light_face_stride, int batch,
                           float* radiance, void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t relight_workspace_bytes(int faces, int k_face, int batch);

/* ---------------------------------------------------------------------------------------------
 * relight_vertices_shifted -- fused per-vertex shift + relight:
 *   radiance[v] = < S_{shift_v} L , T_v >, the shift applied identically to every face.
 *
 * Defines:  P:513 (per pixel, coefficients rotated by the normal's azimuth and elevation),
 *           P:514 (coarser levels by the recursive h_s / h_t filters).
 *
 *   transfer       [num_vertices][faces*N*N] fp32 (full pyramids per face, 64-bit indexing).
 *   faces          1 .. HS_MAX_FACES.
 *   light          [faces][N*N] fp32, one pyramid per face.
 *   vertex_shifts  DEVICE pointer [num_vertices][2] fp32 (sy, sx), finite.
 *   radiance       [num_vertices] fp32, must not overlap transfer, light or vertex_shifts.
 *   workspace      >= relight_shifted_workspace_bytes(...) bytes.
 * Paths: N <= 128 residue planes of the light (exact: the box shift is four integer rolls and the
 * bottom-up commutes with even rolls, so every output level is a rolled read of planes built once
 * per call from the light's fp64 fields); larger N the chunked tile shift + row dot.
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status relight_vertices_shifted(const float* transfer, int64_t num_vertices, int faces,
                                   const float* light, int log2n, const float* vertex_shifts,
                                   float* radiance, void* workspace, size_t workspace_bytes,
                                   void* stream);

HS_API size_t relight_shifted_workspace_bytes(int64_t num_vertices, int faces, int log2n);

/* ---------------------------------------------------------------------------------------------
 * relight_vertices_sparse -- relight with sparse (top-K) transfer vectors.
 *
 * Defines:  P:240-245 (non-linear wavelet approximation: keep the largest coefficients of the
 *           transfer), eq:tripleSum P:253-266 with C_{ij0} = delta_ij: the double product
 *           over the kept coefficients only.
 *
 *   radiance[v][b] = sum_{k < k_sparse} values[v][k] * light[b][indices[v][k]]
 *   indices       DEVICE [num_vertices][k_sparse] int32 in [0, total_coeffs) (duplicates add).
 *   values        DEVICE [num_vertices][k_sparse] fp32.
 *   light         DEVICE [batch][total_coeffs] fp32 (e.g. full shifted pyramids, faces concatenated).
 *   radiance      DEVICE [num_vertices][batch] fp32, no overlap with the inputs or workspace;
 *                 8-byte aligned when batch >= 64 (float2 stores), 4-byte otherwise.
 *   workspace     >= relight_sparse_workspace_bytes(total_coeffs, batch): the light transposed to
 *                 coefficient-major [total_coeffs][batch] (one contiguous row per gathered index).
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status relight_vertices_sparse(const int32_t* indices, const float* values, int64_t num_vertices,
                                         int k_sparse, const float* light, int64_t total_coeffs, int batch,
                                         float* radiance, void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t relight_sparse_workspace_bytes(int64_t total_coeffs, int batch);

/* Seeded sparse transfer rows, bit-identical to synth.sparse_transfer_rows (input generator):
 * per vertex the first faces * 4^dense_levels pairs are every face's levels < dense_levels, the
 * rest hash-drawn detail coefficients; values u * 2^-level (|u| for scaling).                   */
HS_API hs_status hs_fill_sparse_transfer(int32_t* indices, float* values, int64_t row_start, int64_t row_count,
                                         int faces, int log2n, int k_sparse, int dense_levels, uint64_t seed,
                                         void* stream);

/* ---------------------------------------------------------------------------------------------
 * relight_vertices_triple -- triple-product relight, BRDF and visibility separate (SURVEY.md
 * §8(f) f3).
 *
 * Defines:  eq:tripleSum P:253-266  R = sum_ijk C_ijk a_i b_j c_k  with a = light, b = BRDF,
 *           c = visibility and C_ijk the integral of three basis functions, evaluated through the
 *           Tripling Coefficient Theorem P:287-294 (cases (a), (b), (c)); per face:
 *
 *   radiance[v][b] = sum_f  integral over the unit square of  L_bf * rho_vf * V_vf
 *
 *   with every function truncated to its HAAR1 prefix of k_face = 4^k coefficients (levels < k).
 *   brdf_q, vis_q  DEVICE [num_vertices][faces * k_face] fp32 in the qtree layout
 *                  (haar_pack_qtree below).
 *   light          DEVICE [batch][faces][light_face_stride] fp32 in HAAR1 order (the first k_face
 *                  entries of each face are used -- e.g. the band written by haar_shift_coeffs).
 *   radiance       DEVICE [num_vertices][batch] fp32, no overlap with the inputs or workspace;
 *                  16-byte aligned on the tensor-core path (batch % 64 == 0), 4-byte otherwise.
 *   k_face         4^k with 3 <= k <= 12.
 *   workspace      >= relight_triple_workspace_bytes(...), 1024-byte aligned (HS_ERR_ALIGNMENT).
 *   Precision: fp32 inputs; the tripling terms are formed in fp32 and multiplied on the tensor
 *   cores in split fp16 (hi + 2^-11 lo) with fp32 accumulation when batch % 64 == 0 (DESIGN.md
 *   §5.8), each row's terms scaled by a power of two first and rows that leave fp16's range
 *   recomputed exactly on the CUDA cores, as in relight_vertices (any fp32 magnitude of BRDF and
 *   visibility whose tripling terms stay finite), otherwise on CUDA cores in fp32.
 *
 * haar_pack_qtree -- HAAR1 -> qtree layout (the storage format of brdf_q / vis_q):
 *   in   DEVICE [rows][faces][in_face_stride] fp32, HAAR1 prefix of 4^log2k used per face;
 *   out  DEVICE [rows][faces][4^log2k] fp32.  With r = log2k - 3, face f of row v is 4^r chunks
 *   of 64: chunk c (level-r cell (ci, cj) = (c >> r, c & (2^r - 1))) holds, for q = 0..3 (child
 *   cell (2ci + q/2, 2cj + q%2) at level r+1) and p = 0..3 (grandchild (2i1 + p/2, 2j1 + p%2) at
 *   level r+2): slot 15q + 3p + t = grandchild coefficient of type t (H, V, D); slot 15q + 12 + t
 *   = child coefficient of type t; slot 60 + t = coefficient of cell c itself at level r; slot 63
 *   = the mean of the function over cell c (scaling + the coarser levels evaluated on c).  The
 *   layout holds the same information as the HAAR1 prefix (the 4^r cell means determine the
 *   levels < r).  log2k >= 3; in and out must not overlap.
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status relight_vertices_triple(const float* brdf_q, const float* vis_q, int64_t num_vertices, int faces,
                                         int k_face, const float* light, int64_t light_face_stride, int batch,
                                         float* radiance, void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t relight_triple_workspace_bytes(int64_t num_vertices, int faces, int k_face, int batch);

HS_API hs_status haar_pack_qtree(const float* in, int64_t rows, int faces, int64_t in_face_stride, int log2k,
                                 float* out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * relight_vertices_brdf_rotated -- the paper's shading composed (SURVEY.md §8(f) f1 + f3):
 *   R[v][b] = integral over the lat-long map of  L_b * Rot(theta_v, phi_v) rho * V_v,
 * band-limited to the HAAR1 prefix of 4^log2k coefficients, where rho is ONE BRDF map in the local
 * frame of the surface (pole = normal) rotated per vertex by its normal's elevation and azimuth
 * ("rotate the BRDF by the normal's angles, then the triple
 * integral"; R28) -- haar_rotate_coeffs(rho, (alpha, beta) = (theta_v, phi_v)), then
 * haar_pack_qtree, then relight_vertices_triple, chunked over 4096 vertices, all on the device.
 *   brdf          DEVICE [N*N] fp32 HAAR1 pyramid of the local-frame BRDF (N = 2^log2n, lat-long:
 *                 rows theta in [0, pi] top first, columns phi in [0, 2 pi)).
 *   normals_host  HOST [num_vertices][2] fp64 (theta_N, phi_N) radians.
 *   vis_q         DEVICE [num_vertices][4^log2k] fp32 visibility bands in the qtree layout
 *                 (haar_pack_qtree of their HAAR1 prefixes).
 *   light         DEVICE [batch][light_stride] fp32: each frame's HAAR1 prefix of >= 4^log2k
 *                 entries (a full pyramid, stride N*N, or a band, stride 4^log2k); stride % 4 == 0.
 *   radiance      DEVICE [num_vertices][batch] fp32 (16-byte aligned when batch % 64 == 0).
 *   log2n 3 .. 11, log2k 3 .. log2n, batch 1 .. 1024; workspace >= relight_brdf_rotated_workspace_bytes,
 *   1024-byte aligned.
 *   Accuracy: the triple product as relight_vertices_triple; the rotation is the paper's first-order
 *   chain rule (haar_rotate_coeffs), so against the spatial rotation the radiance is approximate
 *   (PSNR, rising with N).
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status relight_vertices_brdf_rotated(const float* brdf, int log2n, const double* normals_host,
                                               int64_t num_vertices, const float* vis_q, int log2k,
                                               const float* light, int64_t light_stride, int batch,
                                               float* radiance, void* workspace, size_t workspace_bytes,
                                               void* stream);

HS_API size_t relight_brdf_rotated_workspace_bytes(int log2n, int log2k, int batch);

/* ---------------------------------------------------------------------------------------------
 * haar_rotate_coeffs -- rotation of lat-long maps directly on their Haar coefficients (SURVEY.md
 * §8(f) f1; the paper's "non-linear phase shift").
 *
 * Defines:  P:350-459 (eq:theta/eq:phi P:397-402: g(theta, phi) = f(Theta, Phi); chain rule
 *           eq:pde1-2 P:416-425 on the coefficients' difference fields), recursion to coarser
 *           levels P:466-497/"rotation around the x-axis followed by a simple shifting along
 *           the phi-axis" P:459/P:508.
 *
 *   in, out       DEVICE [batch][N*N] fp32 HAAR1 pyramids of N x N lat-long maps (rows theta in
 *                 [0, pi] top first, columns phi in [0, 2 pi)); in and out must not overlap.
 *   angles_host   HOST [batch][2] fp64: (alpha, beta) radians -- elevation about X with the active
 *                 matrix R_x(alpha) = [[1,0,0],[0,cos,-sin],[0,sin,cos]] applied as
 *                 g(theta, phi) = f(angles of R_x p), then the shift along phi by beta N / (2 pi)
 *                 columns (f'(x) = f(x - s), exact, as haar_shift_coeffs).
 *   log2n         1 .. 11.   workspace >= haar_rotate_workspace_bytes(log2n, batch), 16-byte aligned.
 *   Accuracy: the elevation is the paper's first-order chain rule on the finest-level difference
 *   fields with bilinear resampling (R25-R27), computed with fp64 angles and fp64
 *   fields and rounded once to fp32: it equals the fp64 oracle of that algorithm to ~1e-7
 *   relative; against the spatial rotation it is approximate by construction (PSNR, improving
 *   with N).  alpha = 0 reproduces the input to fp32 rounding and the azimuth part is exact.
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status haar_rotate_coeffs(const float* in, float* out, int log2n, int batch, const double* angles_host,
                                    void* workspace, size_t workspace_bytes, void* stream);

HS_API size_t haar_rotate_workspace_bytes(int log2n, int batch);

/* hs_enable_peer_access -- let kernels launched on the current device load / store the memory of
 * `peer_device` directly (NVLink / NVSwitch), e.g. relight_vertices writing its radiance rows into
 * rank 0's buffer opened through CUDA IPC (the fused relight + gather of SURVEY.md §8(e),
 * DESIGN.md §6).  HS_OK if enabled or already enabled (or peer_device is the current device),
 * HS_ERR_UNSUPPORTED if the devices cannot access each other.                                     */
HS_API hs_status hs_enable_peer_access(int peer_device);

/* ---------------------------------------------------------------------------------------------
 * hs_fill_transfer -- seeded synthetic transfer rows, generated in place (input generator, not
 * part of the method; bit-identical to synth.transfer_rows):
 *   T[v][f*k_face + k] = u * 2^-level(k), u = ((h >> 40) - 2^23) / 2^23,
 *   h = splitmix64(splitmix64(seed + stream * 0xD1B54A32D192ED03) + global_index),
 *   global_index = (row_start + v) * faces * k_face + f * k_face + k; k == 0 entries are |u|.
 *   out [row_count][faces*k_face] device fp32.
 * ------------------------------------------------------------------------------------------- */
HS_API hs_status hs_fill_transfer(float* out, int64_t row_start, int64_t row_count, int faces,
                           int k_face, uint64_t seed, uint64_t stream_id, void* stream);

/* Kernel-launch count of the most recent successful call on this thread (for bench accounting). */
HS_API int hs_last_launch_count(void);

HS_API const char* hs_status_string(hs_status s);
HS_API const char* hs_last_cuda_error(void);
/* ABI version, bumped on any signature change. */
HS_API int hs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HAARSHIFT_H_ */
