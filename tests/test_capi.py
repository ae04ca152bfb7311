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
    assert L.cox_version() == 1


def test_workspace_query_is_host_only():
    L = _lib.load()
    assert L.cox_permute_workspace_bytes(262144, 8) >= 4 * 2 * 1024 * 8
    assert L.cox_permute_workspace_bytes(0, 8) > 0


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
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path
