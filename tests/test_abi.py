"""The C ABI library loads and exports every symbol include/pspgmres.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pspgmres.h")
SO = os.path.join(ROOT, "paper_1308_5626_b200", "libpspgmres.so")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"\b(psp_[a-z0-9_]+)\s*\(", txt)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ["psp_create", "psp_matvec", "psp_arnoldi_step", "psp_mrep_fit", "psp_precond_apply",
                     "psp_step", "psp_destroy", "psp_solve", "psp_workspace_bytes"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(SO):
        pytest.fail(f"{SO} not built (run make / __graft_entry__.build())")
    lib = ctypes.CDLL(SO)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_1308_5626_b200 import pspgmres
    assert sorted(pspgmres.EXPORTED) == declared_functions()
    lib = pspgmres.lib()
    assert lib.psp_version().decode().startswith("libpspgmres")
    assert lib.psp_status_str(pspgmres.PSP_E_SAMPLES).decode().startswith("insufficient")


def test_create_rejects_bad_arguments_without_gpu():
    # argument validation happens before any device work
    from paper_1308_5626_b200 import pspgmres as P
    lib = P.lib()
    g = P.make_grid((16,))
    s = P.psp_stencil()
    s.kind = P.PSP_OP_CONST_DIFF
    o = P.default_opts()
    nb = ctypes.c_size_t()
    assert lib.psp_workspace_bytes(ctypes.byref(g), ctypes.byref(s), 5, 30, ctypes.byref(o), None,
                                   ctypes.byref(nb)) == P.PSP_E_ARG          # d > 4
    assert lib.psp_workspace_bytes(ctypes.byref(g), ctypes.byref(s), 1, 0, ctypes.byref(o), None,
                                   ctypes.byref(nb)) == P.PSP_E_ARG          # restart < 1
    s.kind = P.PSP_OP_CELL_DIFF
    assert lib.psp_workspace_bytes(ctypes.byref(g), ctypes.byref(s), 1, 30, ctypes.byref(o), None,
                                   ctypes.byref(nb)) == P.PSP_E_ARG          # no field
    g2 = P.make_grid((2,))
    s.kind = P.PSP_OP_CONST_DIFF
    assert lib.psp_workspace_bytes(ctypes.byref(g2), ctypes.byref(s), 1, 30, ctypes.byref(o), None,
                                   ctypes.byref(nb)) == P.PSP_E_DIM          # n < 2d+1


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of psp_grid / psp_stencil / psp_opts / psp_report / psp_mrep_info have
    the C structs' sizes and field offsets (compiled from include/pspgmres.h with gcc)."""
    import shutil
    import subprocess
    from paper_1308_5626_b200 import pspgmres as P
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = [s for s in ("psp_grid", "psp_stencil", "psp_opts", "psp_report", "psp_mrep_info") if hasattr(P, s)]
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HDR}"', "int main(void) {"]
    for s in structs:
        lines.append(f'  printf("{s} size %zu\\n", sizeof({s}));')
        for f, _ in getattr(P, s)._fields_:
            lines.append(f'  printf("{s} {f} %zu\\n", offsetof({s}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            s, f, v = ln.split()
            got[(s, f)] = int(v)
    for s in structs:
        cs = getattr(P, s)
        assert got[(s, "size")] == ctypes.sizeof(cs), s
        for f, _ in cs._fields_:
            assert got[(s, f)] == getattr(cs, f).offset, (s, f)


def test_set_timing_rejects_null_context_without_gpu():
    # psp_set_timing validates before touching a context (bench.py switches levels 1 <-> 2)
    from paper_1308_5626_b200 import pspgmres as P
    lib = P.lib()
    assert lib.psp_set_timing(None, 1) == P.PSP_E_ARG
    assert lib.psp_launch_count(None, None) == P.PSP_E_ARG


def test_comm_selftest_rejects_null_without_gpu():
    from paper_1308_5626_b200 import pspgmres as P
    assert P.lib().psp_comm_selftest(None, None) == P.PSP_E_ARG
