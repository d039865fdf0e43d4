"""CPU-side checks of the C-ABI library: it loads and exports every symbol include/sffn.h declares;
host-only calls (no device compute) behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sffn.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sffn_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_23198_b200 import sffn
    if not os.path.exists(sffn.LIB_PATH):
        import subprocess
        subprocess.check_call(["make", "-C", ROOT, "paper_2603_23198_b200/libsffn.so"])
    return sffn.lib()


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2603_23198_b200 import sffn
    assert set(declared_functions()) == set(sffn._SIGS)


def test_host_only_calls(lib):
    from paper_2603_23198_b200 import sffn
    assert sffn.status_string(0) == "SFFN_OK"
    assert sffn.status_string(3) == "SFFN_ERR_TILE_OVERFLOW"
    assert sffn.twell_words(32768, 14336, 256, 8) == 32768 * 1792
    assert sffn.workspace_bytes(16, 128, 512, 256, 8, "gather") == 16 * 64 * 4 + (1024 - 16 * 64 * 4 % 1024) % 1024
    assert sffn.up_down_workspace_bytes(16, 128, 512, 256, 8, "gather") == 0
    # union workspace: H_c (128 rows per block x N bf16) + the permuted copy of X dominate
    assert sffn.up_down_workspace_bytes(32768, 4096, 14336, 256, 8, "union") >= 256 * 128 * 14336 * 2 + 32768 * 4096 * 2
    assert sffn.workspace_bytes(32768, 4096, 14336, 256, 8) == sffn.workspace_bytes(32768, 4096, 14336, 256, 8, "union")
    assert "sm_100a" in sffn.version()


def test_argument_errors_before_launch(lib):
    """Shape / argument errors are reported on the host without touching a device (none here)."""
    vp = ctypes.c_void_p
    p = vp(4096)  # never dereferenced: validation fails first
    # K % 64 != 0 -> SHAPE
    assert lib.sffn_pack(p, p, 16, 100, 512, 256, 8, p, None, None) == 2
    # bad C -> INVALID_ARG
    assert lib.sffn_pack(p, p, 16, 128, 512, 256, 3, p, None, None) == 1
    # N not a multiple of T -> SHAPE
    assert lib.sffn_pack(p, p, 16, 128, 500, 256, 8, p, None, None) == 2
    # NULL -> INVALID_ARG
    assert lib.sffn_up_down(None, p, p, p, 16, 128, 512, 256, 8, p, None, 0, 1, None) == 1
    # union algo without workspace -> SHAPE
    assert lib.sffn_up_down(p, p, p, p, 16, 128, 512, 256, 8, p, None, 0, 2, None) == 2
    # bad algo -> INVALID_ARG
    assert lib.sffn_up_down(p, p, p, p, 16, 128, 512, 256, 8, p, None, 0, 7, None) == 1
    # misaligned -> INVALID_ARG
    assert lib.sffn_pack(vp(4098), p, 16, 128, 512, 256, 8, p, None, None) == 1
    # workspace too small -> SHAPE
    assert lib.sffn_forward(p, p, p, p, 16, 128, 512, 256, 8, p, p, 10, None, 0, None) == 2


def test_product_path_does_not_import_oracle():
    """The product package must not import, link or call anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2603_23198_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "oracle_" not in s, f


@pytest.mark.parametrize("M,R", [(32768, 8192), (32768, 16384), (32768, 4096), (32768, 2048), (32845, 8192),
                                 (5000, 8192), (100000, 8192), (4096, 8192), (12288, 4096), (1000, 256), (129, 128)])
def test_host_chunk_plan(lib, M, R):
    """sffn_forward_host's chunk schedule: covers M exactly, no chunk above the stage slot (chunk_rows rounded
    to the rows actually staged), chunk starts on the 2048-row permutation windows when chunk_rows allows it,
    and ramps (short first and last chunks: the PCIe pipeline's fill and drain) when there is room."""
    from paper_2603_23198_b200 import sffn
    v = sffn.forward_host_chunks(M, R)
    rows = R if R < M else (M + 127) // 128 * 128
    assert sum(v) == M and all(0 < s <= rows for s in v)
    u = 2048 if R % 2048 == 0 else 128
    starts = [sum(v[:i]) for i in range(len(v))]
    assert all(s0 % u == 0 for s0 in starts)
    if M >= 4 * R and R >= 4096:
        assert v[0] < R and v[-1] < R and max(v) == R
    assert sffn.forward_host_chunks(M, 100) == [] and sffn.forward_host_chunks(0, 128) == []
