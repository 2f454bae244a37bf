"""CPU: the C-ABI library loads and exports every symbol include/fht_b200.h
declares; the host-only helpers match the reference rules.  No GPU compute."""
import re
from pathlib import Path

import oracle
from paper_2411_07351_b200 import _lib, fht

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "fht_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fht_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 21
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.exported_symbols()) == syms
    assert b"sm_100a" in lib.fht_version()


def test_host_helpers_match_oracle():
    for s in (0, 1):
        for w in range(2, 300):
            assert fht.split_width(w, s) == oracle.split_width(w, s)
        for w in (1, 2, 3, 17, 509, 1000, 3001, 8191):
            assert fht.count_additions_tree(w, 5, s) == oracle.count_additions_tree(w, 5, s)
    for num in range(0, 40):
        for den in range(1, 12):
            assert fht.round_half_up_ratio(num, den) == oracle.round_half_up_ratio(num, den)


def test_host_helper_errors():
    import pytest

    with pytest.raises(fht.InvalidArgument):
        fht.split_width(1)
    with pytest.raises(fht.InvalidArgument):
        fht.round_half_up_ratio(1, 0)
    with pytest.raises(fht.InvalidArgument):
        fht.round_half_up_ratio(-1, 3)
    with pytest.raises(fht.InvalidArgument):
        fht.strategy_from_string("fast")
