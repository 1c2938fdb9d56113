"""The ctypes mirrors in paper_2507_13522_b200/cm.py have the layout include/cm.h gives
the C compiler: every struct's size and every field's offset, checked by compiling a tiny C
program against the header (gcc, no CUDA needed).  A field added on one side only (the
way cm_info.numa_node was added) fails here instead of corrupting a GPU run."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2507_13522_b200 import cm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRUCTS = [cm.cm_config, cm.cm_layer_table, cm.cm_adamw, cm.cm_sgd, cm.cm_info, cm.cm_shadow_desc]


def _c_layout(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cm.h"', "int main(void) {"]
    for S in STRUCTS:
        n = S.__name__
        lines.append(f'  printf("{n} size %zu\\n", sizeof({n}));')
        for f, _ in S._fields_:
            lines.append(f'  printf("{n} {f} %zu\\n", offsetof({n}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        n, f, v = line.split()
        out[(n, f)] = int(v)
    return out


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    return _c_layout(tmp_path_factory.mktemp("abi"))


@pytest.mark.parametrize("S", STRUCTS, ids=lambda S: S.__name__)
def test_struct_layout_matches_header(S, c_layout):
    n = S.__name__
    assert C.sizeof(S) == c_layout[(n, "size")], n
    for f, _ in S._fields_:
        assert getattr(S, f).offset == c_layout[(n, f)], (n, f)
