"""CPU: the ctypes mirror of include/saberlda.h (tests/abi.py, what an FFI binding declares)
matches the header's struct layouts exactly -- every field's offset and every struct's size,
as gcc lays them out -- so a binding written from the header cannot drift from the library."""
import shutil
import subprocess
from pathlib import Path

import ctypes as C
import pytest

import abi

REPO = Path(__file__).resolve().parent.parent
STRUCTS = {
    "slda_corpus_view": abi.CorpusView,
    "slda_config": abi.Config,
    "slda_iteration_stats": abi.IterationStats,
    "slda_info": abi.Info,
    "slda_kernel_times": abi.KernelTimes,
    "slda_gen_params": abi.GenParams,
}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_mirror_matches_header_layout(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "saberlda.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for field, _ in py._fields_:
            lines.append(f'  printf("{cname} {field} %zu\\n", offsetof({cname}, {field}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(REPO / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            s, f, v = ln.split()
            got[(s, f)] = int(v)
    for cname, py in STRUCTS.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for field, _ in py._fields_:
            assert got[(cname, field)] == getattr(py, field).offset, (cname, field)
