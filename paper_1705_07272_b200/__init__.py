"""B200-native Haar-domain shift + relight (Alnasser & Foroosh, arXiv 1705.07272).

Thin Python binding over the C ABI of libhaarshift.so (include/haarshift.h): argument marshalling
only -- every step of the hot path runs in the library's sm_100a CUDA kernels.  PyTorch provides
device memory and streams.  Function names follow the C ABI:

* ``haar_shift_coeffs``        shifted Haar pyramids, computed in the Haar domain
* ``relight_vertices``         per-vertex transfer inner products (a6)
* ``relight_vertices_shifted`` fused per-vertex shift + relight (a7)
* ``relight_vertices_sparse``  relight with sparse top-K transfer (f2)
* ``relight_vertices_triple``  triple product, BRDF and visibility separate (f3);
  ``haar_pack_qtree`` converts HAAR1 pyramids to its qtree storage layout
* ``haar_shift_coeffs_coarse`` coarse-start shift (f4)
* ``haar_rotate_coeffs``       rotation of lat-long maps in the Haar domain (f1)
* ``relight_vertices_brdf_rotated``  the paper's shading: BRDF rotated per vertex normal (f1), then
  the triple product with light and visibility (f3)
* ``hs_fill_transfer``         seeded synthetic transfer rows generated in place (input generator)

See DESIGN.md for the method, its readings of the paper, layouts and kernels.
"""
from __future__ import annotations

from ._lib import HaarShiftError, load  # noqa: F401
from .api import (  # noqa: F401
    haar_pack_qtree,
    haar_rotate_coeffs,
    haar_rotate_workspace_bytes,
    haar_shift_coarse_workspace_bytes,
    haar_shift_coeffs,
    haar_shift_coeffs_coarse,
    haar_shift_workspace_bytes,
    enable_peer_access,
    hs_fill_sparse_transfer,
    hs_fill_transfer,
    last_launch_count,
    relight_shifted_workspace_bytes,
    relight_vertices,
    relight_workspace_bytes,
    relight_sparse_workspace_bytes,
    relight_vertices_shifted,
    relight_vertices_sparse,
    relight_triple_workspace_bytes,
    relight_vertices_triple,
    relight_brdf_rotated_workspace_bytes,
    relight_vertices_brdf_rotated,
    shift_and_relight,
)

__all__ = [
    "HaarShiftError", "load", "haar_shift_coeffs", "haar_shift_coeffs_coarse", "haar_shift_coarse_workspace_bytes", "haar_shift_workspace_bytes", "hs_fill_transfer",
    "last_launch_count", "relight_shifted_workspace_bytes", "relight_vertices", "relight_workspace_bytes", "relight_vertices_shifted",
    "shift_and_relight", "hs_fill_sparse_transfer", "relight_vertices_sparse",
    "relight_sparse_workspace_bytes", "haar_pack_qtree", "relight_triple_workspace_bytes", "relight_vertices_triple",
    "haar_rotate_coeffs", "haar_rotate_workspace_bytes", "enable_peer_access",
    "relight_vertices_brdf_rotated", "relight_brdf_rotated_workspace_bytes",
]
