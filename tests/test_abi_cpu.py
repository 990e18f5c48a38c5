"""Host-side checks of the C ABI that need no GPU: the library builds for sm_100a, loads,
exports every symbol include/rici.h declares, validates arguments before touching a device,
and the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2007_02306_b200 import build as b
    b.build()
    from paper_2007_02306_b200 import _lib
    return _lib.load()


def _declared():
    txt = open(os.path.join(ROOT, "include", "rici.h")).read()
    return sorted(set(re.findall(r"RICI_API[^;]*?\b(rici_\w+)\s*\(", txt, re.S)))


def test_header_symbols_exported(lib):
    declared = _declared()
    assert len(declared) == 16
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2007_02306_b200", "librici.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (rici_\w+)", out))
    assert set(declared) <= exported
    for name in declared:
        assert hasattr(lib, name)


def test_kernel_timing_api(lib):
    import ctypes
    ms, n = ctypes.c_float(1.0), ctypes.c_int64(7)
    assert lib.rici_kernel_time_ms(5, ctypes.byref(ms), ctypes.byref(n)) == 1        # unknown id
    assert lib.rici_kernel_time_ms(0, None, None) == 1                               # null outputs
    assert lib.rici_kernel_time_ms(1, ctypes.byref(ms), ctypes.byref(n)) == 0
    assert n.value == 0 and ms.value == 0.0                                          # nothing recorded
    assert lib.rici_set_kernel_timing(0) == 0


def test_sass_is_sm100a():
    so = os.path.join(ROOT, "paper_2007_02306_b200", "librici.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_argument_validation(lib):
    assert lib.rici_version().decode().startswith("rici-b200")
    P = ctypes.c_void_p
    # null mesh / bad sizes are rejected synchronously, before any device work
    assert lib.rici_generate(None, None, 0, ctypes.c_float(0.3), 64, None, None) == 1
    h = P()
    assert lib.rici_create_mesh(None, -1, None, 0, None, ctypes.byref(h)) == 1
    assert b"negative" in lib.rici_last_error()
    assert lib.rici_crss_search(None, 5, None, 5, 64, None, None) == 1
    assert lib.rici_crss_search(P(1), 6, P(1), 5, 64, P(1), None) == 1      # n_haystack < n_needles
    assert lib.rici_crss_pairs(P(1), 1, P(1), 1, 1, P(1), 1, P(1), None) == 1  # n_bins < 2
    assert lib.rici_crss_distances(P(1), 1, P(1), 1, 129, P(1), None) == 1    # n_bins > 128
    assert lib.rici_create_mesh(P(1), 3, P(1), (1 << 28) + 1, None, ctypes.byref(h)) == 1   # > max triangles
    assert b"triangles" in lib.rici_last_error()
    assert lib.rici_crss_search_ex(P(1), 1, P(1), 1, 64, 8, P(1), None) == 1                 # unknown flag
    assert lib.rici_clutter_fraction(None, None, None, 0, ctypes.c_float(0.3), 4, None, None, None) == 1
    assert lib.rici_destroy_mesh(None) == 0
    assert lib.rici_mesh_num_triangles(None) == -1
    assert lib.rici_crss_guard_stats(None, 0) == 1                                           # null out


def test_product_does_not_touch_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline may use oracle/: the
    package and the scripts never import it."""
    for dirpath, _, files in [w for d in ("paper_2007_02306_b200", "scripts") for w in os.walk(os.path.join(ROOT, d))]:
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "librici_oracle" not in txt and "rici_oracle.c" not in txt, f
                assert not re.search(r"#include\s*[<\"].*oracle", txt), f


def test_bench_reference_arm_prints_contract_line():
    """bench.py --impl reference runs the oracle on the host (no GPU) and prints one JSON line."""
    import json
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "images/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
