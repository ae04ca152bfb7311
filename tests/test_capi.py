"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import re
from pathlib import Path

from paper_2605_17889_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "coxmoe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(cox_\w+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_symbols() == set(_lib.EXPORTS)


def test_library_exports_all_symbols():
    L = _lib.load()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert L.cox_version() == _lib.ABI_VERSION == 3


def test_workspace_query_is_host_only():
    L = _lib.load()
    assert L.cox_permute_workspace_bytes(262144, 8) >= 4 * 2 * 1024 * 8
    assert L.cox_permute_workspace_bytes(0, 8) > 0
    # router: zeroed header for the decode tickets + T*E + T fp32 scratch (tensor-core screen)
    assert L.cox_router_workspace_bytes(262144, 64) >= 4 * (262144 * 64 + 262144)
    assert L.cox_router_workspace_bytes(0, 8) >= 512


def test_argument_validation_is_host_only():
    """Invalid arguments are rejected before any device work (no GPU needed):
    expert ids must name a segment of offsets[E+1]; the router needs its workspace."""
    import ctypes
    L = _lib.load()
    ids = (ctypes.c_int32 * 2)(0, 8)
    ptrs = (ctypes.c_void_p * 2)(4096, 8192)
    rc = L.cox_grouped_swiglu(4096, 100, 4096, 8, 2, ids, ptrs, 256, 256, 4096, 0, None)
    assert rc == _lib.COX_EINVAL and b"outside [0, 8)" in L.cox_last_error()
    ids[1] = -1
    rc = L.cox_grouped_down(4096, 100, 4096, 8, 2, ids, ptrs, 256, 256, 4096, 0, None)
    assert rc == _lib.COX_EINVAL
    rc = L.cox_router_topk(4096, _lib.DTYPE_BF16, 4096, _lib.DTYPE_BF16, 64, 256, 8, 2, 0, 4096, 4096, 4096,
                           4096, 16, None)
    assert rc == _lib.COX_EINVAL and b"workspace" in L.cox_last_error()
    # K3 gather mode: needs row_tokens, d % 64 == 0, expert ids inside [0, E)
    ids[1] = 3
    rc = L.cox_grouped_swiglu_gather(4096, 100, None, 4096, 8, 2, ids, ptrs, 256, 256, 4096, 0, None)
    assert rc == _lib.COX_EINVAL and b"row_tokens" in L.cox_last_error()
    rc = L.cox_grouped_swiglu_gather(4096, 100, 4096, 4096, 8, 2, ids, ptrs, 96, 256, 4096, 0, None)
    assert rc == _lib.COX_EINVAL and b"d%64" in L.cox_last_error()
    ids[1] = 9
    rc = L.cox_grouped_swiglu_gather(4096, 100, 4096, 4096, 8, 2, ids, ptrs, 256, 256, 4096, 0, None)
    assert rc == _lib.COX_EINVAL and b"outside [0, 8)" in L.cox_last_error()


def test_sass_contains_tcgen05_and_tma():
    """The built library carries sm_100a tensor-core (UTCHMMA) and TMA (UTMALDG) code."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        import pytest
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "LDGSTS" in sass and "FHFMA" in sass  # K3 gather mode (cp.async), mixed-precision re-score FMAs
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path
