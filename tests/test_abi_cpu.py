"""CPU-side checks of the boundary: the C-ABI library builds, loads without a GPU,
and exports every symbol include/*.h declares; no compute calls."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libmod():
    from paper_2405_16267_b200 import build
    build.build()
    from paper_2405_16267_b200 import bicadmm
    bicadmm.lib()
    return bicadmm


def _declared():
    names = set()
    for h in ("bicadmm.h", "bicadmm_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(bicadmm_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol(libmod):
    decl = _declared()
    assert len(decl) >= 20
    L = libmod.lib()
    for name in sorted(decl):
        assert hasattr(L, name), name
    assert set(libmod.ABI_SYMBOLS) == decl


def test_version_and_rc_strings(libmod):
    L = libmod.lib()
    assert L.bicadmm_version() == 1
    assert L.bicadmm_rc_string(-3) == b"label outside the loss domain"
    assert L.bicadmm_uid_size() >= 128


def test_sm100a_sass_present():
    # the .so carries sm_100a SASS (not only PTX) for the hot kernels
    import subprocess
    so = os.path.join(ROOT, "paper_2405_16267_b200", "libbicadmm.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in sass           # FP64 tensor-core Gram
    assert "LDG.E.ENL2.128" in sass or "LDG.E.128" in sass or "LDG.E.EL.128" in sass or ".128" in sass


def test_validation_errors_without_gpu(libmod):
    # argument validation happens before any device call
    import ctypes as ct
    import numpy as np
    bc = libmod
    m = np.array([10], dtype=np.int64)
    cs = np.array([0, 8], dtype=np.int64)
    blk = (bc.bicadmm_block * 1)(bc.bicadmm_block(0, 0, 16, 8))
    bptr = (ct.c_void_p * 1)(16)
    P = bc.bicadmm_problem(1, 1, 1, bc.LS, bc.F64, 1, 8, m.ctypes.data_as(ct.POINTER(ct.c_int64)),
                           cs.ctypes.data_as(ct.POINTER(ct.c_int64)), blk, bptr)
    n = ct.c_size_t(0)
    good = bc.Params(kappa=2).struct()
    assert bc.lib().bicadmm_workspace_size(ct.byref(P), ct.byref(good), ct.byref(n)) == 0 and n.value > 0
    bad = bc.Params(kappa=9).struct()      # kappa > n*C
    assert bc.lib().bicadmm_workspace_size(ct.byref(P), ct.byref(bad), ct.byref(n)) == bc.ERR_INVALID
    bad = bc.Params(kappa=2, alpha=1.5).struct()
    assert bc.lib().bicadmm_workspace_size(ct.byref(P), ct.byref(bad), ct.byref(n)) == bc.ERR_INVALID
    cs2 = np.array([0, 6], dtype=np.int64)  # col_start must end at n
    P.col_start = cs2.ctypes.data_as(ct.POINTER(ct.c_int64))
    assert bc.lib().bicadmm_workspace_size(ct.byref(P), ct.byref(good), ct.byref(n)) == bc.ERR_DIM
    P.col_start = cs.ctypes.data_as(ct.POINTER(ct.c_int64))
    blk[0].lda = 6                           # lda not a multiple of 4
    assert bc.lib().bicadmm_workspace_size(ct.byref(P), ct.byref(good), ct.byref(n)) == bc.ERR_INVALID


def test_product_path_does_not_import_oracle():
    # the product package never imports, links or calls the oracle
    pkg = os.path.join(ROOT, "paper_2405_16267_b200")
    bad = re.compile(r"(^\s*(from|import)\s+oracle)|liborc|\borc_[a-z]|orc\.h", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not bad.search(src), f


def test_ctypes_struct_layout_matches_header(tmp_path):
    # the binding's ctypes structs against the C header: size and every field offset, read
    # from a tiny gcc-compiled program (a drifted field would silently corrupt the ABI)
    import ctypes as ct
    import subprocess
    from paper_2405_16267_b200 import bicadmm as bc
    structs = [bc.bicadmm_block, bc.bicadmm_problem, bc.bicadmm_params, bc.bicadmm_step_info, bc.bicadmm_report]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "bicadmm.h"', 'int main(void) {']
    for S in structs:
        name = S.__name__
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for f in S._fields_:   # ctypes names a C field `lambda` as `lambda_`
            lines.append(f'printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0].rstrip("_")}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for S in structs:
        name = S.__name__
        assert got[(name, "size")] == ct.sizeof(S), name
        for f in S._fields_:
            assert got[(name, f[0])] == getattr(S, f[0]).offset, (name, f[0])


def test_binding_argument_counts_match_prototypes():
    # every prototype in include/*.h against the binding's argtypes (count per function)
    import ctypes as ct
    from paper_2405_16267_b200 import bicadmm as bc
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    protos = {}
    for h in ("bicadmm.h", "bicadmm_ops.h"):
        text = open(os.path.join(root, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
        for m in re.finditer(r"\b(bicadmm_\w+)\s*\(([^;{]*?)\)\s*;", text):
            args = m.group(2).strip()
            protos[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    L = bc.lib()
    checked = 0
    for name, n in protos.items():
        f = getattr(L, name, None)
        if f is None or f.argtypes is None:
            continue
        assert len(f.argtypes) == n, (name, len(f.argtypes), n)
        checked += 1
    assert checked >= 20, checked
