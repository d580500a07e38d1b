"""CPU oracle for the Haar-domain shift + relight hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The product path
(``paper_1705_07272_b200``) never imports it, and the oracle imports nothing from the product:
the two share no code; only ``synth`` (seeded input generators, none of the method's arithmetic)
serves both.

What it computes (DESIGN.md §2 lists every reading of the paper):

* ``haar``:   unit-square orthonormal 2D non-separable (quadtree) Haar and unit-interval 1D Haar,
  forward and inverse, HAAR1 packing.
* ``shift``:  the shifted pyramid by the paper's own ground-truth procedure (PAPER.md P:535:
  "rotating it in the spatial domain to generate the ground truth"): inverse transform, pixel
  shift by box projection ("linear shift"), forward transform.
* ``relight``: the double product R = T . L'  (PAPER.md eq:tripleSum P:265-266 with the Tripling
  Coefficient Theorem's scaling case P:287: C_{i j 0} = delta_ij) and the per-vertex
  fused form r_v = <S_{s_v} L, T_v>; the sparse gather and the triple
  product as the pixel-domain triple integral (eq:tripleSum).
* ``rotate``: rotation of lat-long maps by the spatial ground truth: inverse,
  bilinear resampling at the rotated angles (eq:theta/eq:phi P:397-402), the azimuth shift,
  forward; PSNR; and ``rotate_coeffs_chain``, the paper's own (approximate, first-order)
  chain-rule algorithm written stage by stage.  The GPU's rotation is accurate to a PSNR against
  the spatial truth, not to 1e-5 (R25); its 1e-5 agreement with rotate_coeffs_chain is a
  regression check of the kernels.

Everything is fp64 NumPy, written step by step with no blocking, fusion or reordering.
Pins (tests/test_oracle_*.py, "-m 'not gpu'"): SPEC worked examples, dense
basis-matrix brute force built from the basis definition, exact ``fractions.Fraction`` overlap
integrals <psi_i, T_s psi_j> for 1D N=8 and 2D 4x4, closed forms (identity at 0 and N, integer
composition, DC invariance, Parseval, linearity in the fractional part), SURVEY App. B examples.
The rotation's chain-rule stages are pinned one by one (tests/test_oracle_rotate.py): the
recursion against forward2d on exact fields, the closure (identity on exact fields, a strict
improvement toward the analytic rotation), the DC rule's level cap by which levels can move it,
exact cases (identity, constants, integer azimuths, the half turn) and first-order convergence to
the analytic rotation.  Where the paper is silent (the pole rows R26, the closure and the DC rule
R27) those pins fix the READING, not a value the paper prints: the paper gives no worked example
of its rotation, only PSNRs of its own data (Tables 1-4).
"""
from . import haar, shift, relight, rotate  # noqa: F401

__all__ = ["haar", "shift", "relight", "rotate"]
