"""The C-ABI library loads and exports every symbol include/vbddc.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vbddc.h")).read()
    return sorted(set(re.findall(r"^(?:vb_status|const char \*)\s*(vb_\w+)\(", src, re.M)))


def test_library_exports_header_symbols():
    import paper_2304_09770_b200 as vb
    lib = ctypes.CDLL(vb.LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(vb.EXPORTED) == names


def test_error_paths_without_context():
    import paper_2304_09770_b200 as vb
    lib = ctypes.CDLL(vb.LIB_PATH)
    lib.vb_factor.argtypes = [ctypes.c_void_p]
    assert lib.vb_factor(None) == vb.VB_EINVAL
    lib.vb_destroy.argtypes = [ctypes.c_void_p]
    assert lib.vb_destroy(None) == vb.VB_EINVAL


def test_debug_gemm_argument_checks_without_gpu():
    """vb_debug_gemm rejects non-positive sizes and short leading dimensions before any device work."""
    import paper_2304_09770_b200 as vb
    f = vb._vb_debug_gemm
    dummy = ctypes.c_void_p(16)
    # M = 0
    assert f(0, 4, 4, 1.0, dummy, 4, 0, dummy, 4, 0, None, 0.0, dummy, 4, 1, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
    # lda < M (A not transposed)
    assert f(8, 4, 4, 1.0, dummy, 4, 0, dummy, 4, 0, None, 0.0, dummy, 8, 1, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
    # ldb < N (B transposed)
    assert f(8, 6, 4, 1.0, dummy, 8, 0, dummy, 4, 1, None, 0.0, dummy, 8, 1, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
    # ldc < M
    assert f(8, 4, 4, 1.0, dummy, 8, 0, dummy, 4, 0, None, 0.0, dummy, 4, 1, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
    # null C / batch 0
    assert f(8, 4, 4, 1.0, dummy, 8, 0, dummy, 4, 0, None, 0.0, None, 8, 1, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
    assert f(8, 4, 4, 1.0, dummy, 8, 0, dummy, 4, 0, None, 0.0, dummy, 8, 0, 0, 0, 0, None, 0, 0, 0) == vb.VB_EINVAL
