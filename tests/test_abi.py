"""The C-ABI library loads and exports every symbol include/zkl.h declares (CPU only, no compute)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "zkl.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zkl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ["zkl_tlookup_prepare", "zkl_tlookup_prove", "zkl_sumcheck_prove", "zkl_table_create",
                 "zkl_vec_import", "zkl_vec_export", "zkl_ctx_create", "zkl_workspace_bytes"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2404_16109_b200 import build, zkl
    lib_path = build.build()
    L = ctypes.CDLL(lib_path)          # loads without a GPU (CUDA runtime is linked statically)
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (zkl_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert set(zkl.EXPORTED) == set(declared_symbols())


def test_workspace_sizing_host_logic():
    from paper_2404_16109_b200 import zkl
    L = zkl.lib()
    assert L.zkl_workspace_bytes(3, 4, 1) == 0            # not a power of two
    small = L.zkl_workspace_bytes(1 << 10, 1 << 8, 1)
    big = L.zkl_workspace_bytes(1 << 26, 1 << 16, 1)
    assert 0 < small < big
    # the D-side buffers dominate at scale: A + fold ping-pong ~ 3 x 32 B per local element
    assert big >= (1 << 26) * 32 * 2
    assert L.zkl_table_bytes(1 << 16) >= (1 << 16) * 32
    assert L.zkl_strerror(5) == b"lookup not in table"
