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
