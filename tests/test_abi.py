"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/ecmg.h declares;
without a GPU it refuses to create a grid (no CPU fallback). No GPU needed."""
import ctypes as C
import os
import re
import subprocess

import pytest

import __graft_entry__ as ge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ecmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ecmg_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    return ge.build_lib()


def test_header_declares_the_six_calls():
    syms = declared_symbols()
    for s in ("ecmg_create_grid", "ecmg_set_coeffs", "ecmg_solve_level", "ecmg_prolongate_extrapolate",
              "ecmg_richardson", "ecmg_run", "ecmg_destroy_grid", "ecmg_strerror"):
        assert s in syms


def test_exports_every_declared_symbol(libpath):
    L = C.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_built_for_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_names_match_abi():
    from paper_1506_02983_b200 import ecmg
    for s in declared_symbols():
        assert s in ecmg.EXPORTS
        assert callable(getattr(ecmg, s[len("ecmg_"):]))


def test_strerror_and_no_gpu_behaviour(libpath):
    import torch
    from paper_1506_02983_b200 import ecmg
    assert ecmg.strerror(ecmg.ENOTCONV).startswith("JCG")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    st, h = ecmg.create_grid((0, 0, 0), (1, 1, 1), (4, 4, 4), 4)
    assert st == ecmg.ECUDA and not h.value   # no CPU fallback


def test_invalid_arguments(libpath):
    from paper_1506_02983_b200 import ecmg
    st, h = ecmg.create_grid((0, 0, 0), (1, 1, 1), (4, 4, 4), 2)     # fewer than 3 levels
    assert st == ecmg.EINVAL
    st, h = ecmg.create_grid((0, 0, 0), (0, 1, 1), (4, 4, 4), 4)     # empty extent
    assert st == ecmg.EINVAL
    assert ecmg.lib().ecmg_destroy_grid(None) == ecmg.EINVAL


def test_struct_layouts_match_header(tmp_path):
    # the ctypes mirrors of the ABI structs (ecmg.py) have the header's sizes and field offsets (compiled with gcc)
    import ctypes as C
    import subprocess
    from paper_1506_02983_b200 import ecmg as E
    structs = {"ecmg_problem": E.ecmg_problem, "ecmg_stats": E.ecmg_stats, "ecmg_box": E.ecmg_box,
               "ecmg_dist": E.ecmg_dist}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "ecmg.h"', "int main(void) {"]
    for name, cls in structs.items():
        src.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            src.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)], text=True).splitlines())
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_binding_option_ids_match_the_header():
    # every ECMG_OPT_* of include/ecmg.h has the same value in the Python binding, and the binding names no other
    from paper_1506_02983_b200 import ecmg
    src = open(os.path.join(ROOT, "include", "ecmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    hdr = {m.group(1): int(m.group(2)) for m in re.finditer(r"\bECMG_(OPT_[A-Z_0-9]+)\s*=\s*(\d+)", src)}
    assert len(hdr) >= 20 and len(set(hdr.values())) == len(hdr)
    py = {k: v for k, v in vars(ecmg).items() if k.startswith("OPT_")}
    assert py == hdr
