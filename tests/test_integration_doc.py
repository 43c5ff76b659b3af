"""INTEGRATION.md's reference-side ctypes stub stays in step with the ABI (CPU).

The stub is what a fdroof maintainer would paste into pkg/src/fdroof/b200.py;
its argument struct must have the size the library was compiled with, and the
ABI version it sends must be the library's.
"""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_source() -> str:
    with open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8") as fh:
        text = fh.read()
    m = re.search(r"```python\n(# pkg/src/fdroof/b200\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its ctypes stub"
    return m.group(1)


def test_stub_struct_matches_library():
    from paper_1608_03984_b200 import _lib

    src = _stub_source()
    cls = re.search(r"(class _Args\(ctypes\.Structure\):.*?\])[^\n]*\n", src, re.S).group(1)
    ns = {"ctypes": ctypes}
    exec(cls, ns)  # noqa: S102 -- the documented struct, nothing else
    lib = _lib.load()
    assert ctypes.sizeof(ns["_Args"]) == lib.fdr_acoustic_args_size()


def test_stub_sends_the_library_abi_version():
    src = _stub_source()
    assert "abi_version=_lib.fdr_abi_version()" in src
