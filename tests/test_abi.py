"""C ABI checks that need no GPU: the library builds/loads and exports every
function include/*.h declares; argument validation that fails before any
device work (null pointers, bad n) returns the documented codes."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        src = re.sub(r"//[^\n]*", "", src)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b([A-Za-z_]\w*)\s*\(", src, flags=re.M):
            name = m.group(1)
            if name not in ("if", "while", "return", "sizeof"):
                names.append(name)
    return sorted(set(names))


def lib():
    import paper_2205_11659_b200 as tb
    return tb.load()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("paren_match", "tree_bbox", "tb_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    L = lib()
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, f"libtreebbox.so lacks {missing}"


def test_host_checkable_errors():
    L = lib()
    assert L.paren_match(None, 0, None, None, None) == 0          # n == 0: no-op
    assert L.paren_match(None, -1, None, None, None) == -1        # n < 0
    assert L.paren_match(None, 1 << 31, None, None, None) == -1   # n > 2^31-1
    assert L.paren_match(None, 10, None, None, None) == -1        # null pointers
    assert b"null" in L.tb_last_error()
    assert L.tree_bbox(None, None, 0, None, None) == 0
    assert L.tree_bbox(None, None, 5, None, None) == -1
    assert L.paren_match_workspace_bytes(0) == 0


def test_shared_object_is_sm100a():
    so = os.path.join(ROOT, "paper_2205_11659_b200", "libtreebbox.so")
    lib()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
