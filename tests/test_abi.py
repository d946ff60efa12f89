"""The C-ABI library loads on a CPU-only host and exports exactly what
include/fsgpu.h declares; the ctypes mirror of fs_plan matches the C layout.
No compute call is made (there is no GPU here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_1506_08620_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "fsgpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int|int64_t|size_t|uint64_t|void|fs_gate\s*\*)\s*(fs_\w+)\s*\(", text, flags=re.M)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s+(fs_\w+)$", nm, flags=re.M))
    assert set(declared_functions()) <= exported


def test_version_and_workspace():
    lib = _lib.load()
    assert b"sm_100a" in lib.fs_version()
    assert lib.fs_workspace_bytes() >= 64


def test_library_built_from_these_sources():
    # fs_version() embeds the hash of the sources + nvcc flags it was built from
    import __graft_entry__ as g

    assert _lib.load().fs_version().decode().split()[-2:] == ["src", g.source_sha16()]


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_without_gpu():
    """Invalid arguments are rejected before any CUDA call (ValueError contract)."""
    lib = _lib.load()
    pos = ctypes.c_int64(-1)
    assert lib.fs_certify(0, None, 4, 16, 1, None, None, None, None, None, ctypes.byref(pos), None) == _lib.FS_INVALID_ARG
    assert b"qbits" in lib.fs_last_error()
    assert lib.fs_certify(0, None, 4, 32, 0, None, None, None, None, None, ctypes.byref(pos), None) == _lib.FS_INVALID_ARG
    plan = _lib.FsPlan()
    plan.algorithm = 99
    plan.dtype = 0
    plan.n1 = 4
    plan.x = 1
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, None, None) == _lib.FS_INVALID_ARG
    plan.algorithm = _lib.ALGO_CODES["direct"]
    plan.table = 1
    plan.q = 1
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 3, 1, None) == _lib.FS_INVALID_ARG
    assert b"out_bytes" in lib.fs_last_error()
    plan.algorithm = _lib.ALGO_CODES["direct-cache"]
    plan.q = 2
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
    # optional accelerators whose extents would index outside their tables
    plan.algorithm = _lib.ALGO_CODES["direct"]
    plan.q = 1
    plan.r = 1000  # directory of (1000 >> 5) + 1 = 32 words
    plan.rank = 1
    plan.hot_word0, plan.hot_words, plan.hot_knot0, plan.hot_knots = 30, 5, 0, 2
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
    assert b"hot window" in lib.fs_last_error()
    plan.hot_word0, plan.hot_words, plan.hot_knot0, plan.hot_knots = 0, 32, 3, 2  # knots past n1 = 4
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
    plan.hot_words = 0
    plan.sparse = 1
    for shift, ndense in ((4, 0), (17, 0), (5, 40)):
        plan.sparse_shift, plan.sparse_ndense = shift, ndense
        assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
        assert b"sparse" in lib.fs_last_error()
    # group records: shifts 5..14 only; unknown formats rejected
    plan.sparse_format = _lib.SPARSE_RECORDS
    for shift, novf in ((4, 0), (15, 0), (5, 40)):
        plan.sparse_shift, plan.sparse_ndense = shift, novf
        assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
        assert b"sparse" in lib.fs_last_error()
    plan.sparse_format, plan.sparse_shift, plan.sparse_ndense = 10, 8, 0
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
    assert b"sparse" in lib.fs_last_error()
    # knot bytes: one per knot, beside the gap-1 rank directory
    plan.sparse_format, plan.sparse_shift, plan.sparse_ndense = _lib.SPARSE_KNOT_BYTES, 0, 3  # n1 = 4
    assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
    assert b"knot bytes" in lib.fs_last_error()
    # count words: one stripe shift 0..27 for the table
    plan.sparse_format = _lib.SPARSE_COUNT
    for shift in (-1, 28):
        plan.sparse_shift = shift
        assert lib.fs_search_device(ctypes.byref(plan), None, 0, None, 4, 1, None) == _lib.FS_INVALID_ARG
        assert b"count-word" in lib.fs_last_error()
    cb = lib.fs_count_words_bytes
    assert cb(1000, 0, 0) == 8 * 63 and cb(1000, 6, 0) == 8 and cb(1000, 27, 0) == 8 and cb(1000, 28, 0) == 0
    assert cb(1 << 32, 3, 0) == 0 and cb(1000, 6, 4) == 8 + 16 and cb(1000, 9, 4) == 0  # offsets: bytes, k <= 8
    rb = lib.fs_sparse_rec_bytes
    assert rb(_lib.SPARSE_RECORDS, 4, 1000, 15, 0) == 0 and rb(_lib.SPARSE_RECORDS, 4, 1000, 5, 0) == 16 * 33
    assert rb(_lib.SPARSE_RECORDS8, 4, 1000, 5, 0) == (8 * 33 + 15) // 16 * 16
    assert rb(_lib.SPARSE_RECORDS8, 4, 1000, 5, 2) == (8 * 33 + 2 * 4 + 15) // 16 * 16
    assert rb(_lib.SPARSE_TWO_LEVEL, 4, 1000, 5, 0) == 0 and rb(5, 4, 1000, 5, 0) == 0
    assert rb(_lib.SPARSE_RECORDS8X3, 4, 1000, 11, 0) == 16 and rb(_lib.SPARSE_RECORDS8X3, 4, 1000, 12, 0) == 0
    assert rb(_lib.SPARSE_RECORDS12, 4, 1000, 10, 0) == 16 * 2 and rb(_lib.SPARSE_RECORDS12, 4, 1000, 11, 0) == 0


def test_status_codes_map_to_reference_exceptions():
    import paper_1506_08620_b200 as fs

    with pytest.raises(fs.NotDistinguishable) as e:
        _lib.check(_lib.FS_NOT_DISTINGUISHABLE, pos=2)
    assert e.value.position == 2
    with pytest.raises(fs.Overflow):
        _lib.check(_lib.FS_OVERFLOW)
    with pytest.raises(fs.OutOfDomain) as e:
        _lib.check(_lib.FS_OUT_OF_DOMAIN, pos=7)
    assert e.value.position == 7
    with pytest.raises(ValueError):
        _lib.check(_lib.FS_INVALID_ARG)
    with pytest.raises(ValueError):
        _lib.check(_lib.FS_INCONSISTENT)
    with pytest.raises(fs.DeviceError):
        _lib.check(_lib.FS_CUDA_ERROR)


def test_fs_plan_layout_matches_c(tmp_path):
    fields = [f for f, _ in _lib.FsPlan._fields_]
    src = tmp_path / "layout.c"
    body = "\n".join(f'  printf("{f} %zu\\n", offsetof(fs_plan, {f}));' for f in fields)
    src.write_text(
        "#include <stdio.h>\n#include <stddef.h>\n#include \"fsgpu.h\"\n"
        "int main(void) {\n  printf(\"sizeof %zu\\n\", sizeof(fs_plan));\n" + body + "\n  return 0;\n}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if line)
    assert int(out["sizeof"]) == ctypes.sizeof(_lib.FsPlan)
    for f in fields:
        assert int(out[f]) == getattr(_lib.FsPlan, f).offset, f


def test_integration_stub_matches_c_layout():
    """The maintainer-side ctypes stub printed in INTEGRATION.md declares the
    same fs_plan as the library (field names, types and offsets)."""
    text = (ROOT / "INTEGRATION.md").read_text()
    block = text.split("class fs_plan(ctypes.Structure):")[1].split("]\n", 1)[0] + "]"
    ns = {"ctypes": ctypes}
    exec("class fs_plan(ctypes.Structure):" + block, ns)
    stub = ns["fs_plan"]
    assert [f for f, _ in stub._fields_] == [f for f, _ in _lib.FsPlan._fields_]
    assert ctypes.sizeof(stub) == ctypes.sizeof(_lib.FsPlan)
    for f, _ in stub._fields_:
        assert getattr(stub, f).offset == getattr(_lib.FsPlan, f).offset, f
