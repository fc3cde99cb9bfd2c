"""CPU checks of the C ABI library: it builds for sm_100a, loads, and exports
every entry point include/stkde.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1705_09366_b200 import build
    return build.build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "stkde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stkde_\w+)\s*\(", src)))


def test_header_declares_expected_calls():
    names = declared_functions()
    for must in ("stkde_plan_create", "stkde_compute", "stkde_compute_sharded", "stkde_compute_slab",
                 "stkde_plan_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    L = ctypes.CDLL(lib_path)
    for name in declared_functions():
        assert hasattr(L, name), name
    from paper_1705_09366_b200 import EXPORTS
    assert sorted(EXPORTS) == declared_functions()


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_strerror_without_gpu(lib_path):
    from paper_1705_09366_b200 import load_library
    L = load_library(lib_path)
    assert L.stkde_strerror(0) == b"ok"
    assert b"max_n" in L.stkde_strerror(-4)


def test_product_does_not_import_oracle():
    # the product package must never reach the oracle (test infrastructure only)
    pkg = os.path.join(ROOT, "paper_1705_09366_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "stkde_oracle" not in txt and "liboracle" not in txt, f


def test_phase_names_and_nccl_id_without_gpu(lib_path):
    # host-only calls: the phase names of stkde_plan_phase_ms and the NCCL unique id
    import paper_1705_09366_b200 as S
    L = S.load_library(lib_path)
    assert tuple(L.stkde_phase_name(i).decode() for i in range(len(S.PHASES))) == S.PHASES
    assert L.stkde_phase_name(len(S.PHASES)) is None and L.stkde_phase_name(-1) is None
    assert b"NCCL" in L.stkde_strerror(S.STKDE_ENCCL)
    try:
        uid = S.nccl_unique_id()
    except S.StkdeError as e:            # no NCCL in this process: the documented error
        assert e.code == S.STKDE_ENCCL
        return
    assert len(uid) == 128 and uid != S.nccl_unique_id()
