"""C-ABI: the library loads on CPU, exports every symbol include/glucosim.h
declares, and the ctypes structures match the C layouts (sizeof/offsetof
computed by compiling the header with gcc).  No compute calls."""

import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "glucosim.h")
SO = os.path.join(REPO, "paper_2202_13927_b200", "libglucosim.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(SO):
        subprocess.run(["make", "-C", os.path.join(REPO, "paper_2202_13927_b200", "csrc"), "-s", "-j4"],
                       check=True)
    return C.CDLL(SO)


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+\**(gt_\w+)\s*\(", txt, flags=re.M)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    from paper_2202_13927_b200 import _lib
    assert sorted(s[0] for s in _lib.SIGNATURES) == names


def test_abi_version(lib):
    lib.gt_abi_version.restype = C.c_int
    assert lib.gt_abi_version() == 3


def test_struct_layouts_match_c():
    from paper_2202_13927_b200 import _lib
    structs = {"gt_parity_args": _lib.ParityArgs, "gt_fast_args": _lib.FastArgs,
               "gt_reduce_args": _lib.ReduceArgs, "gt_sampler_args": _lib.SamplerArgs,
               "gt_meal_gen": _lib.MealGen, "gt_northern_args": _lib.NorthernArgs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'printf("{cname}.{f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", src, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = dict(l.rsplit(" ", 1) for l in out.strip().splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f in py._fields_:
            assert int(got[f"{cname}.{f[0]}"]) == getattr(py, f[0]).offset, f"{cname}.{f[0]}"


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2202_13927_b200 import engine, _lib
    with pytest.raises(_lib.GlucosimError):
        engine.require_device()
