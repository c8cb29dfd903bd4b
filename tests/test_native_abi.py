"""CPU-side checks of the C ABI: the library loads and exports every symbol the
header declares; no compute calls (no GPU here)."""

import os
import re

from paper_1909_05098_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fedheat_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fh_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_match_binding_list():
    assert declared() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = N.lib()
    for name in declared():
        assert hasattr(L, name), name


def test_status_codes_match_header():
    from paper_1909_05098_b200 import errors
    text = open(HEADER).read()
    for name in ("FH_OK", "FH_ERR_CONFIG", "FH_ERR_INSTABILITY", "FH_ERR_DEVICE", "FH_ERR_DEGENERATE"):
        val = int(re.search(rf"#define {name} (\d+)", text).group(1))
        assert getattr(errors, name) == val


def test_version_and_device_count_without_gpu():
    L = N.lib()
    assert L.fh_version() == 1
    assert N.device_count() >= 0
