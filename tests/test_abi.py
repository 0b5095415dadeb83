"""The C-ABI library loads without a GPU and exports every entry point that
include/pic_b200.h declares; the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pic_b200.h")
LIB = os.path.join(ROOT, "paper_2102_13133_b200", "libpic_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(pic_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pic_context_create", "pic_advance_p", "pic_load_interpolators", "pic_unload_currents",
                 "pic_advance_b", "pic_advance_e", "pic_ghost_sync_fields", "pic_ghost_fold_currents",
                 "pic_sort_particles", "pic_step", "pic_step_host", "pic_species_upload", "pic_last_error"):
        assert must in names
    assert len(names) >= 35


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    lib.pic_version.restype = ctypes.c_int
    assert lib.pic_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_kernels_are_the_cuda_path():
    """The default push (advance_p_lean, variant 52) is real sm_100a SASS:
    TMA bulk copies of the particle slices, vector reductions into the
    accumulator, no local-memory traffic; the sort ranks with MATCH."""
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    # the default in-place form: kOrd = 0, packed FP32 (kPk = 1)
    push = [f for f in funcs
            if f.startswith("_ZN4picb14advance_p_leanILi8ELi6ELb0ELb0ELi0ELi4ELi0ELb0ELb1ELi0ELb0ELi0ELb1E")]
    assert push, "default advance_p kernel not found"
    body = push[0]
    assert "REDG.E.ADD.F32x4" in body
    assert "UBLKCP" in body  # cp.async.bulk (TMA) slice loads / stores
    assert "LDL" not in body and "STL" not in body  # no spills
    assert "FFMA2" in body and "FADD2" in body  # packed FP32 push arithmetic
    scatter = [f for f in funcs if "radix_scatter_kernel" in f.split("\n", 1)[0]]
    assert scatter and any("MATCH" in f for f in scatter)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2102_13133_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text), f"{fn} references the oracle"
