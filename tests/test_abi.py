"""CPU-side checks of the C-ABI boundary (-m "not gpu"): the library builds for
sm_100a, loads, exports every function include/sr_sort.h declares, and rejects
bad arguments before touching a device."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1609_04471_b200 as sr
from paper_1609_04471_b200 import build as srbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "sr_sort.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sr_[a-z_]+)\s*\(", txt)))


def test_header_declares_expected_entry_points():
    fns = _header_functions()
    assert fns == sorted(sr.EXPORTS)


def test_library_exports_every_declared_symbol():
    path = srbuild.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for f in _header_functions():
        assert f in syms, f
    L = sr.lib()
    for f in _header_functions():
        assert hasattr(L, f)


def test_checked_library_exports_and_checks():
    """The checked build (-DSR_CHECKED: device-side SR_CHECK index asserts, the
    stand-in for compute-sanitizer on this pool) exports the same symbols and
    contains the trap the normal build does not."""
    path = srbuild.build(checked=True)
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for f in _header_functions():
        assert f in syms, f
    traps = lambda p: subprocess.check_output(["cuobjdump", "-sass", p], text=True).count("BPT.TRAP")
    assert traps(path) > traps(srbuild.build())


def test_sass_is_sm100a():
    path = srbuild.build()
    out = subprocess.check_output(["cuobjdump", "--list-elf", path], text=True)
    assert "sm_100a" in out


def test_status_strings():
    L = sr.lib()
    assert L.sr_status_string(0) == b"ok"
    assert L.sr_status_string(3) == b"size out of range"


@pytest.mark.parametrize("args,code", [
    ((None, -1, 0, None), 1),          # n < 0
    ((None, 10, 7, None), 2),          # dtype
    ((None, 2**31, 0, None), 3),       # too large
    ((None, 10, 0, None), 1),          # NULL with n >= 2
    ((ctypes.c_void_p(2), 10, 0, None), 4),  # misaligned int32 pointer
    ((ctypes.c_void_p(4), 10, 1, None), 4),  # misaligned int64 pointer
    ((None, 0, 0, None), 0),           # n == 0: no-op
    ((None, 1, 0, None), 0),           # n == 1: no-op
])
def test_sort_keys_argument_errors(args, code):
    assert sr.lib().sr_sort_keys(*args) == code


def test_sort_pairs_argument_errors():
    L = sr.lib()
    assert L.sr_sort_pairs(ctypes.c_void_p(16), None, 10, 0, None) == 1
    assert L.sr_sort_pairs(ctypes.c_void_p(16), ctypes.c_void_p(2), 10, 0, None) == 4
    assert L.sr_sort_pairs(None, None, 1, 0, None) == 0


def test_set_option_validation():
    L = sr.lib()
    assert L.sr_set_option(0, 99) == 1
    assert L.sr_set_option(42, 0) == 1
    assert L.sr_set_option(0, 0) == 0
    assert L.sr_last_plan(None) == 1


def test_step_entry_argument_errors():
    L = sr.lib()
    assert L.sr_tile_sort(ctypes.c_void_p(16), None, 100, 0, 9000, None) == 1   # tile > kCap
    assert L.sr_splitters(ctypes.c_void_p(16), 100, 0, 3, None, None, None, None) == 1
    assert L.sr_presort_scan(ctypes.c_void_p(16), 100, 5, 0, 4096, None, None, 0, None) == 2
