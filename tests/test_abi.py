"""The C ABI library loads and exports every symbol include/dpkfac.h declares,
and the ctypes mirrors have the C struct layouts (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dpkfac.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dpk_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2206_15143_b200 import _lib

    lib = _lib.load()
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert set(declared) == set(_lib.EXPORTED)
    assert b"sm_100a" in lib.dpk_version()


def test_struct_layouts_match_header(tmp_path):
    from paper_2206_15143_b200 import _lib as L

    names = {"dpk_operand": L.Operand, "dpk_factor_job": L.FactorJob, "dpk_gemm_job": L.GemmJob,
             "dpk_pi_job": L.PiJob, "dpk_spd_job": L.SpdJob, "dpk_precond_job": L.PrecondJob,
             "dpk_eig_job": L.EigJob, "dpk_segment": L.Segment, "dpk_spd_factor_job": L.SpdFactorJob,
             "dpk_precond_factor_job": L.PrecondFactorJob, "dpk_im2col_job": L.Im2colJob}
    prog = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname in names:
        prog.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
    prog += ['printf("off_sn %zu\\n", offsetof(dpk_operand, sn));', "return 0;}"]
    c = tmp_path / "sizes.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], check=True, capture_output=True,
                                                       text=True).stdout.splitlines())
    for cname, cls in names.items():
        assert int(out[cname]) == ctypes.sizeof(cls), cname
    assert int(out["off_sn"]) == L.Operand.sn.offset


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2206_15143_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "/root/reference" not in text, f
