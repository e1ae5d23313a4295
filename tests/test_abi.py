"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import os
import re

from paper_1606_09218_b200 import _native

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_functions():
    text = open(os.path.join(ROOT, "include", "rs_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = _native.load_library()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)
    assert lib.rs_abi_version() == 1


def test_workspace_queries_without_gpu():
    lib = _native.load_library()
    assert lib.rs_syrk_workspace_bytes(256, 700) > 0
    assert lib.rs_core_workspace_bytes(12, 12, 12, 1000, 14) >= 12 ** 3 * 8
    assert lib.rs_assemble_workspace_bytes(256, 4, 12, 50, 14, 3) >= 4 * 256 * (12 + 50 * 14) * 8
    assert lib.rs_sum_workspace_bytes(1000) >= 16
    # Tucker-only planes: 96 < r3 <= 160 reserves the slices of the Ozaki-split tcgen05 GEMM
    if os.environ.get("RSB200_TUCKER_OZ", "7") in ("6", "7"):
        base = 4 * 256 * 132 * 8
        with_oz = lib.rs_assemble_workspace_bytes(256, 4, 132, 0, 0, 1)
        assert with_oz >= base + lib.rs_oz_workspace_bytes(4 * 256, 256, 132, 7)
        assert lib.rs_assemble_workspace_bytes(256, 4, 96, 0, 0, 1) < with_oz


def test_domain_errors_without_gpu():
    lib = _native.load_library()
    # argument validation happens before any launch
    assert lib.rs_syrk(None, 3, 4, 3, None, None, 0, None) == 1
    assert b"even" in lib.rs_last_error()
    assert lib.rs_assemble_planes(None, 1, 1, 1, None, None, None, 8, None, None, 99, 1,
                                  None, None, None, None, None, None, 0, 0, 4, 3, None, None, 0,
                                  None) == 1
