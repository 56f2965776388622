"""CPU-side checks of the C-ABI boundary: the library loads without a GPU
and exports every symbol include/mixtera_b200.h declares."""

from __future__ import annotations

import re
from pathlib import Path

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "mixtera_b200.h").read_text()
    return sorted(set(re.findall(r"\b(mx_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    from paper_2502_19790_b200 import _lib

    assert sorted(_lib.EXPORTED) == _declared()


def test_library_loads_and_exports_all_symbols():
    from paper_2502_19790_b200 import _lib, build

    build.build()
    h = _lib.load_library()
    for name in _declared():
        assert hasattr(h, name), name
    assert h.mx_abi_version() == 2
