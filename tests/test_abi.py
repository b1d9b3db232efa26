"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol include/turboreg.h
declares, the binding's struct layouts match the header, and the product package never touches oracle/."""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "turboreg.h")
PKG = os.path.join(ROOT, "paper_2507_01439_b200")


@pytest.fixture(scope="module")
def lib():
    from paper_2507_01439_b200.build import build

    build()
    import paper_2507_01439_b200 as p

    return p.library()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(turboreg_[a-z_]+)\s*\(", text)))


def test_header_declares_the_north_star_entry_points():
    fns = declared_functions()
    for f in ("turboreg_create", "turboreg_register", "turboreg_register_batch", "turboreg_destroy"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in declared_functions():
        assert hasattr(lib, f), f
    out = os.popen(f"nm -D --defined-only {lib._name}").read()
    for f in declared_functions():
        assert re.search(rf"\bT {f}\b", out), f


def test_status_strings_without_gpu(lib):
    assert lib.turboreg_status_string(0) == b"ok"
    assert lib.turboreg_status_string(5) == b"no hypothesis"


def test_create_fails_cleanly_without_gpu_or_bad_args(lib):
    import paper_2507_01439_b200._binding as b

    h = ctypes.c_void_p()
    bad = b.Params(-1.0, 0.0, 10, 2, 0.1, 0, 0)
    assert lib.turboreg_create(ctypes.byref(bad), 0, 100, 1, ctypes.byref(h)) == 1  # invalid argument, no launch
    good = b.Params(0.01, 0.0, 10, 2, 0.1, 0, 0)
    assert lib.turboreg_create(ctypes.byref(good), 0, 2, 1, ctypes.byref(h)) == 1  # max_n < 3
    assert lib.turboreg_register(None, None, None, 0, None) == 1


def test_result_layout_matches_header(lib):
    import paper_2507_01439_b200._binding as b

    assert ctypes.sizeof(b.Result) == 104
    assert ctypes.sizeof(b.Params) == 28
    assert b.Result.num_edges.offset == 96 and b.Result.status.offset == 80


def test_kernels_are_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {lib._name} 2>&1").read()
    assert "sm_100a" in out


def test_product_package_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                continue
            src = open(os.path.join(dirpath, f)).read()
            if f.endswith(".py"):
                tree = ast.parse(src)
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
            else:
                assert "turboreg_oracle" not in src and "oracle_" not in src, f


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_2507_01439_b200._binding as b

    monkeypatch.setattr(b, "_LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(b, "_lib", None)
    with pytest.raises(ImportError):
        b.library()


def test_parameter_validation_without_gpu(lib):
    import paper_2507_01439_b200._binding as b

    h = ctypes.c_void_p()
    # (tau, tau_base, k1, k2, thr, graph_mode, flags): every case is rejected before any CUDA call
    cases = [
        (0.01, 0.0, 10, 2, 0.1, 2, 0),                                  # unknown graph mode
        (0.01, 0.0, 10000, 2, 0.1, 1, 0),                               # SC^2 mode above the canonical-sort cap
        (0.01, 0.0, 10, 2, 0.1, 0, b.F_RANK_MAE | b.F_RANK_MSE),        # two ranking metrics
        (0.01, 0.0, 10, 2, 0.1, 0, 0x100),                              # unknown flag
        (0.01, 0.005, 10, 2, 0.1, 0, 0),                                # tau_base below tau
        (0.01, 0.0, 10, 0, 0.1, 0, 0),                                  # k2 < 1
        (0.01, 0.0, 10, 2, 0.0, 0, 0),                                  # inlier threshold <= 0
    ]
    for c in cases:
        prm = b.Params(*c)
        assert lib.turboreg_create(ctypes.byref(prm), 0, 100, 1, ctypes.byref(h)) == 1, c
