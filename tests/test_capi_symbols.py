"""The C-ABI library loads without a GPU and exports every symbol that
include/treeattn_b200.h declares (no compute calls)."""
import ctypes
import os
import re

from paper_2404_00242_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "treeattn_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ta_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_what_binding_expects():
    assert declared() == sorted(capi.EXPORTED)


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(capi.LIB_PATH)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert capi.lib().ta_abi_version() == 2


def test_no_oracle_linkage():
    """The product library must not depend on the oracle / reference harness."""
    data = open(capi.LIB_PATH, "rb").read()
    for needle in (b"liboracle", b"libtreeattn_ref", b"to_partition_flatten", b"ref_run_iteration"):
        assert needle not in data
