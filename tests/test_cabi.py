"""The drop-in boundary: libopara.so loads and exports every symbol the
public header declares (no device calls)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

from paper_2312_10351_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "opara.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(opara_[a-z_0-9]+)\(", text, re.M)))


def test_header_declares_the_expected_surface():
    syms = declared_symbols()
    for must in ("opara_dag_create", "opara_allocate_streams", "opara_order", "opara_validate_plan",
                 "opara_exec_capture", "opara_exec_replay", "opara_exec_profile", "opara_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib._LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_version_and_error_plumbing():
    L = _lib.lib()
    from paper_2312_10351_b200 import __version__, build
    v = L.opara_version().decode()
    assert v.startswith(__version__ + " sm_100a")
    # provenance: the loaded binary was built from exactly the sources in the tree
    assert v.rpartition("src:")[2] == build.source_hash()
    h = ctypes.c_void_p()
    st = L.opara_dag_create(None, -1, None, 0, ctypes.byref(h))
    assert st == 8 and b"bad arguments" in L.opara_last_error()
