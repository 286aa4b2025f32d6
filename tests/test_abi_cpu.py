"""The C ABI library without a GPU: it loads, exports every symbol include/appd.h
declares, and its host-only calls behave (no compute calls are made here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "appd.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2407_07058_b200 import build as B

    B.build()  # nvcc cross-compiles for sm_100a without a GPU
    import paper_2407_07058_b200 as P

    return P.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(appd_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("appd_create", "appd_solve_weights", "appd_solve_points", "appd_destroy"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_status_strings_and_version(lib):
    assert lib.appd_status_string(0) == b"APPD_OK"
    assert lib.appd_status_string(3) == b"APPD_ERR_NOT_SYMMETRIC"
    assert lib.appd_status_string(42) == b"APPD_ERR_UNKNOWN"
    assert b"sm_100a" in lib.appd_version()


def test_row_ranges_partition_rows(lib):
    import paper_2407_07058_b200 as P

    for n in (1, 5, 127, 128, 129, 1000, 4096, 65536, 131072, 100003):
        for world in (1, 2, 3, 4, 8):
            blocks = [P.appd_row_range_of(n, r, world) for r in range(world)]
            nxt = 0
            for r0, rows in blocks:
                assert r0 == nxt and rows >= 0
                assert r0 % 128 == 0 or rows == 0
                nxt = r0 + rows
            assert nxt == n
    r0, rows = ctypes.c_int64(), ctypes.c_int64()
    assert lib.appd_row_range_of(10, 2, 2, ctypes.byref(r0), ctypes.byref(rows)) == 1  # rank >= world


def test_options_defaults_and_create_without_gpu(lib):
    import paper_2407_07058_b200.binding as B

    o = B.appd_options()
    lib.appd_options_init(ctypes.byref(o))
    assert o.struct_size == ctypes.sizeof(B.appd_options)
    assert (o.world, o.validate, o.sense, o.variant) == (1, 1, 1, 0)
    h = ctypes.c_void_p()
    status = lib.appd_create(ctypes.byref(h), ctypes.byref(o))
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert status == 7 and not h.value  # APPD_ERR_CUDA, no context
    else:
        lib.appd_destroy(h)
    bad = B.appd_options()
    lib.appd_options_init(ctypes.byref(bad))
    bad.struct_size = 3
    assert lib.appd_create(ctypes.byref(h), ctypes.byref(bad)) == 1
    lib.appd_options_init(ctypes.byref(bad))
    bad.variant = 3  # variants are 0 (AUTO), 1 (PRIM), 2 (BORUVKA)
    assert lib.appd_create(ctypes.byref(h), ctypes.byref(bad)) == 1
    lib.appd_options_init(ctypes.byref(bad))
    bad.timeout_ms = -1
    assert lib.appd_create(ctypes.byref(h), ctypes.byref(bad)) == 1
    lib.appd_options_init(ctypes.byref(bad))
    bad.world, bad.rank = 2, 0  # world > 1 needs an NCCL id or a host exchange callback
    assert lib.appd_create(ctypes.byref(h), ctypes.byref(bad)) == 1
    lib.appd_options_init(ctypes.byref(bad))
    bad.metric = 3  # metrics are 0, 1, 2
    assert lib.appd_create(ctypes.byref(h), ctypes.byref(bad)) == 1
    lib.appd_destroy(None)  # NULL-safe


def test_nccl_unique_id_without_gpu(lib):
    import paper_2407_07058_b200 as P

    try:
        a = P.appd_get_nccl_unique_id()
    except P.AppdError as e:  # no usable network interface in this sandbox
        pytest.skip(str(e))
    assert len(a) == 128


def test_binding_refuses_cpu_fallback():
    """The product path has no CPU fallback: a missing library raises."""
    import paper_2407_07058_b200.binding as B

    with pytest.raises(OSError):
        B.load.__wrapped__("/nonexistent/libappd.so") if hasattr(B.load, "__wrapped__") else _load_fresh(
            "/nonexistent/libappd.so")


def _load_fresh(path):
    import importlib

    import paper_2407_07058_b200.binding as B

    saved = B._lib
    try:
        B._lib = None
        return B.load(path)
    finally:
        B._lib = saved
        importlib.invalidate_caches()


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of appd_options / appd_stats have the C header's size and field
    offsets (gcc compiles a probe against include/appd.h)."""
    import subprocess

    import paper_2407_07058_b200.binding as B

    probe = tmp_path / "probe.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "appd.h"', "int main(void) {"]
    for struct, cls in (("appd_options", B.appd_options), ("appd_stats", B.appd_stats)):
        lines.append(f'printf("{struct} size %zu\\n", sizeof({struct}));')
        for name, _ in cls._fields_:
            lines.append(f'printf("{struct} {name} %zu\\n", offsetof({struct}, {name}));')
    lines += ["return 0; }"]
    probe.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {}
    for line in out:
        if line:
            st, name, val = line.split()
            got[(st, name)] = int(val)
    for struct, cls in (("appd_options", B.appd_options), ("appd_stats", B.appd_stats)):
        assert got[(struct, "size")] == ctypes.sizeof(cls), struct
        for name, _ in cls._fields_:
            assert got[(struct, name)] == getattr(cls, name).offset, (struct, name)
