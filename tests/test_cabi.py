"""CPU-side checks of the C ABI boundary: the shared library loads and exports every
symbol include/tmstore.h declares (no compute calls — there is no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tmstore.h")
LIB = os.path.join(ROOT, "paper_2508_11553_b200", "libtmstore.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tm_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_expected_api():
    syms = declared_symbols()
    for s in ["tm_store_create", "tm_record_batch", "tm_match_batch", "tm_export_rows", "tm_session_stats",
              "tm_session_rows", "tm_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []


def test_python_binding_covers_header():
    from paper_2508_11553_b200._lib import SIGNATURES

    assert sorted(SIGNATURES) == declared_symbols()


def test_version_string(lib):
    lib.tm_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.tm_version()


def test_store_create_fails_loudly_without_gpu(lib):
    """No CPU fallback: creating a store with no usable GPU returns an error code."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = lib.tm_store_create(None, ctypes.byref(h))
    assert rc != 0
    lib.tm_last_error.restype = ctypes.c_char_p
    assert lib.tm_last_error()


def declared_arities():
    """tm_* name -> parameter count, from the prototypes in include/tmstore.h."""
    src = re.sub(r"/\*.*?\*/", " ", open(HEADER).read(), flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tm_\w+)\s*\(([^;{]*?)\)\s*;", src, re.M):
        params = " ".join(m.group(2).split())
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_python_binding_arities_match_header():
    """Every ctypes signature in _lib.SIGNATURES passes as many arguments as the C
    prototype takes (a mismatch would only show up as a crash on the GPU box)."""
    from paper_2508_11553_b200._lib import SIGNATURES

    ar = declared_arities()
    assert sorted(ar) == declared_symbols()
    bad = {k: (len(SIGNATURES[k][1]), ar[k]) for k in ar if len(SIGNATURES[k][1]) != ar[k]}
    assert bad == {}


def _ctype_of(param: str):
    p = " ".join(param.split())
    if "*" in p:
        return "ptr"
    for c_name, kind in (("uint64_t", "u64"), ("int64_t", "i64"), ("uint32_t", "u32"), ("int32_t", "i32"),
                         ("double", "f64"), ("int", "i32")):
        if re.search(r"\b" + c_name + r"\b", p):
            return kind
    raise AssertionError(f"unmapped C parameter type: {param!r}")


def test_python_binding_types_match_header():
    """...and in every position the same kind of argument: pointer, int32, int64 (an int32 /
    int64 swap would pass ctypes and corrupt the call)."""
    import ctypes as C

    from paper_2508_11553_b200._lib import SIGNATURES

    kind = {C.c_void_p: "ptr", C.c_char_p: "ptr", C.c_int64: "i64", C.c_int32: "i32", C.c_int: "i32",
            C.c_uint64: "u64", C.c_uint32: "u32", C.c_double: "f64"}
    src = re.sub(r"/\*.*?\*/", " ", open(HEADER).read(), flags=re.S)
    bad = []
    for m in re.finditer(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tm_\w+)\s*\(([^;{]*?)\)\s*;", src, re.M):
        params = [x for x in m.group(2).split(",") if x.strip() and x.strip() != "void"]
        want = [_ctype_of(x) for x in params]
        got = [kind.get(t, repr(t)) for t in SIGNATURES[m.group(1)][1]]
        if want != got:
            bad.append((m.group(1), want, got))
    assert bad == []


def test_python_constants_match_header_enums():
    """Status codes, memory kinds, row orders and profiler kernel kinds: the Python side's
    numbers are the header's."""
    from paper_2508_11553_b200 import _lib
    from paper_2508_11553_b200.store import DeviceStore

    src = re.sub(r"/\*.*?\*/", " ", open(HEADER).read(), flags=re.S)
    enums = {k: int(v) for k, v in re.findall(r"\b(TM_[A-Z0-9_]+)\s*=\s*(\d+)", src)}
    for name in ("TM_OK", "TM_EINVAL", "TM_ENOENT", "TM_ENOMEM", "TM_ECUDA", "TM_MEM_HOST", "TM_MEM_DEVICE",
                 "TM_ORDER_INSERT", "TM_ORDER_LEX"):
        assert getattr(_lib, name) == enums[name], name
    kernels = {k[len("TM_KERNEL_"):].lower(): v for k, v in enums.items() if k.startswith("TM_KERNEL_")}
    assert DeviceStore.KERNELS == kernels
