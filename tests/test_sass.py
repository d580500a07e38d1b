"""The built library is Blackwell-native where it claims to be (-m "not gpu"; cuobjdump only):
the tensor-core relights issue tcgen05.mma (UTCHMMA) with TMEM loads / stores (LDTM / STTM) fed by
TMA (UTMALDG), the fused per-vertex path is the residue-plane kernels, and no kernel falls back to
the legacy HMMA / Hopper HGMMA paths (B200_PROFILING.md, "What proves a Blackwell-native kernel")."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1705_07272_b200", "lib", "libhaarshift.so")
sys.path.insert(0, os.path.join(ROOT, "scripts"))


@pytest.fixture(scope="module")
def counts():
    if shutil.which("cuobjdump") is None or not os.path.exists(LIB):
        pytest.skip("cuobjdump or the built library is not available")
    import sass_evidence
    return {sass_evidence.short(k): v for k, v in sass_evidence.kernel_counts(LIB).items()}


@pytest.mark.parametrize("kernel", ["relight_tc_kernel", "relight_triple_tc_kernel"])
def test_tensor_core_kernels_are_tcgen05(counts, kernel):
    c = counts[kernel]
    assert c["UTCHMMA"] > 0 and c["LDTM"] > 0 and c["STTM"] > 0 and c["UTMALDG"] > 0


def test_no_legacy_tensor_paths(counts):
    assert all(c["HMMA"] == 0 and c["HGMMA"] == 0 for c in counts.values())


def test_fused_per_vertex_path_is_the_residue_planes(counts):
    names = set(counts)
    assert {"planes_kernel", "planes3_kernel", "planes_a_kernel", "planes_c_kernel", "small_planes_kernel"} <= names
    assert any(k.startswith("small_relight_kernel") for k in names)
