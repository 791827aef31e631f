"""libcszi.so loads on CPU-only hosts and exports every symbol include/cszi.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "cszi.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cszi_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2312_05492_b200 import _lib

    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    # the binding binds exactly the declared surface
    assert sorted(_lib.EXPORTED) == names


def test_abi_struct_sizes_match_binding():
    from paper_2312_05492_b200 import _lib

    lib = _lib.load()
    sizes = (ctypes.c_uint64 * 4)()
    lib.cszi_abi_sizes(sizes)
    assert tuple(sizes) == (ctypes.sizeof(_lib.Geom), ctypes.sizeof(_lib.Params),
                            ctypes.sizeof(_lib.Caps), ctypes.sizeof(_lib.Ctl))
    assert b"sm_100a" in lib.cszi_version()


def test_library_is_sm100a_cubin():
    import subprocess

    from paper_2312_05492_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        return  # cuobjdump unavailable
    assert "sm_100a" in out.stdout


def test_workspace_queries_are_host_only():
    from paper_2312_05492_b200 import _lib
    from paper_2312_05492_b200.predictor import default_layout, make_geom

    lib = _lib.load()
    g = make_geom((512, 512, 512), default_layout(3))
    caps = _lib.Caps(bits_cap=1 << 20, outlier_cap=1 << 10)
    ws = lib.cszi_compress_workspace_size(ctypes.byref(g), 512, ctypes.byref(caps))
    assert ws > 2 * 512 ** 3
    cap = lib.cszi_payload_capacity(ctypes.byref(g), 512, ctypes.byref(caps))
    assert cap > 4 * 65 ** 3 + 1024
