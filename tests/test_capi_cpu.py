"""CPU-side checks of the boundary: the C-ABI library loads without a GPU and
exports every symbol include/kvp_b200.h declares (no compute calls here)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "kvp_b200.h").read_text()
    return sorted(set(re.findall(r"\b(kvp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_23914_b200 import _capi
    lib = _capi.lib()
    names = declared_symbols()
    assert names, "no symbols parsed from the header"
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(_capi.SIGNATURES), set(names) - set(_capi.SIGNATURES)
    assert lib.kvp_abi_version() == 1
