"""The C-ABI library loads and exports every entry point `include/lodb200.h` declares
(no compute calls: runs on CPU-only hosts)."""
import os
import re

from paper_2302_14801_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "lodb200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(lod_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_expected_api():
    syms = declared_symbols()
    for s in ("lod_split", "lod_voxelize", "lod_build", "lod_tree_create", "lod_last_error"):
        assert s in syms


def test_library_exports_all_declared_symbols():
    lib = _abi.load(build_if_missing=True)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_table_matches_header():
    assert sorted(n for n, _, _ in _abi.SIGNATURES) == declared_symbols()


def test_version_and_error_without_gpu():
    lib = _abi.load(build_if_missing=True)
    assert b"sm_100a" in lib.lod_version()
    assert lib.lod_last_error() is not None


def test_node_record_layout():
    assert _abi.node_dtype().itemsize == 88
