"""CPU: the C-ABI library loads without a GPU and exports exactly what
include/dbfs.h declares; the Python binding covers every symbol."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dbfs.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(dbfs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "dbfs_bfs" in names and "dbfs_graph_build_rmat" in names and "dbfs_validate" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    from paper_1803_03922_b200 import _lib
    L = _lib.load()
    for name in declared():
        assert hasattr(L, name), name
    assert set(declared()) == set(_lib.SIGNATURES), set(declared()) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_and_abi_version():
    from paper_1803_03922_b200 import _lib
    L = _lib.load()
    assert L.dbfs_abi_version() == 1
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.DeviceUnavailable):
        _lib.Context(0)


def test_struct_sizes_match_header():
    # compile a tiny C probe against the header to compare struct layouts
    import subprocess, tempfile
    from paper_1803_03922_b200 import _lib
    src = r'''
    #include <stdio.h>
    #include <stddef.h>
    #include "dbfs.h"
    int main(void){
      printf("%zu %zu %zu %zu %zu\n", sizeof(dbfs_rmat_params), sizeof(dbfs_graph_info),
             sizeof(dbfs_bfs_options), sizeof(dbfs_run_stats), sizeof(dbfs_iteration));
      return 0; }
    '''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        sizes = [int(x) for x in subprocess.check_output([exe]).split()]
    assert sizes == [ctypes.sizeof(_lib.RmatParamsC), ctypes.sizeof(_lib.GraphInfoC),
                     ctypes.sizeof(_lib.BfsOptionsC), ctypes.sizeof(_lib.RunStatsC),
                     ctypes.sizeof(_lib.IterationC)]
