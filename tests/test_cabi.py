"""The C-ABI library loads and exports every symbol include/conserve_b200.h declares
(no compute calls: runs on CPU)."""
import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "conserve_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2410_01228_b200 import _ffi
    lib = ctypes.CDLL(_ffi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_ffi_table_covers_header():
    from paper_2410_01228_b200 import _ffi
    assert set(declared_symbols()) == set(_ffi.EXPORTS)


def test_version_and_host_only_engine():
    import paper_2410_01228_b200 as cs
    assert b"sm_100a" in cs.lib().cs_version()
    cfg = cs.model_config("tiny", flags=cs._ffi.CS_FLAG_HOST_ONLY)
    with cs.KvPool(cfg) as kv:
        kv.register_request(0, False)
        assert kv.allocate(0, 33).ok
        kv.commit_allocations(0)
        blocks, slots = kv.block_table(0)
        assert blocks == [0, 1, 2] and slots == [-1, -1, -1]
        kv.audit()


def test_config_validation_errors():
    import pytest
    import paper_2410_01228_b200 as cs
    cfg = cs.model_config("tiny", flags=cs._ffi.CS_FLAG_HOST_ONLY, page_tokens=32)
    with pytest.raises(cs.CsConfigError, match="page_tokens is fixed at 16"):
        cs.KvPool(cfg)
    cfg = cs.model_config("tiny", flags=0, kv_bytes_per_token=196608)  # validated before any CUDA call
    with pytest.raises(cs.CsConfigError, match="kv_bytes_per_token"):
        cs.KvPool(cfg)
