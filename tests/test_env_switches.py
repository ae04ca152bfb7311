"""Every environment switch the library or bench reads is documented in
INTEGRATION.md's table (the product runs on defaults; the switches are A/B
experiments and must not sprawl undocumented)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_every_env_switch_is_documented():
    srcs = list((ROOT / "paper_2605_17889_b200" / "csrc").glob("*.c*")) + \
        list((ROOT / "paper_2605_17889_b200").glob("*.py")) + [ROOT / "bench.py"]
    used = set()
    for p in srcs:
        text = p.read_text()
        used |= set(re.findall(r'env_int\("(COX_[A-Z0-9_]+)"', text))
        used |= set(re.findall(r'getenv\("(COX[A-Z0-9_]+)"\)', text))
        used |= set(re.findall(r'environ(?:\.get)?\(?\[?"(COX[A-Z0-9_]+)"', text))
    doc = (ROOT / "INTEGRATION.md").read_text()
    missing = sorted(v for v in used if f"`{v}`" not in doc)
    assert used, "no switches found: the scan is broken"
    assert not missing, f"undocumented environment switches: {missing}"
