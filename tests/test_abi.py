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
    assert lib.gt_abi_version() == 4


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


def _fast_args(**kw):
    from paper_2202_13927_b200 import _lib
    a = _lib.FastArgs()
    a.n, a.dt_s, a.period_s, a.period_steps = 4, 60.0, 300.0, 5
    a.horizon_ticks, a.grid_step_ticks, a.n_days, a.n_grid = 2880, 60, 2, 48
    a.hypo_min_ticks, a.controller = 15, 1
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def _call_fast(lib, a):
    from paper_2202_13927_b200 import _lib
    fn = lib.gt_simulate_fast
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(_lib.FastArgs), C.c_void_p]
    rc = fn(C.byref(a), None)
    buf = C.create_string_buffer(512)
    lib.gt_last_error(buf, C.c_int64(512))
    return rc, buf.value.decode()


@pytest.mark.parametrize("n_days", [1, 3, 0])
def test_fast_rejects_a_day_buffer_that_does_not_match_the_horizon(lib, n_days):
    """Advisor finding r01: the kernels index the day buffers by t // 86400
    without a bound, so n_days must be exactly max(1, ceil(horizon / 1 day));
    the check runs before any CUDA call (works without a GPU)."""
    rc, msg = _call_fast(lib, _fast_args(n_days=n_days))
    assert rc == -1 and "n_days" in msg, (rc, msg)   # GT_EINVAL


def test_parity_rejects_a_short_day_buffer(lib):
    from paper_2202_13927_b200 import _lib
    a = _lib.ParityArgs()
    a.n, a.dt_s, a.period_s, a.period_steps = 2, 30.0, 300.0, 10
    a.horizon_ticks, a.grid_step_ticks, a.n_days, a.n_grid, a.block_ticks = 5760, 120, 1, 48, 5760
    fn = lib.gt_simulate_parity
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(_lib.ParityArgs), C.c_void_p]
    assert fn(C.byref(a), None) == -1


def test_fast_rejects_negative_slice_count(lib):
    rc, msg = _call_fast(lib, _fast_args(n_slices=-3))
    assert rc == -1 and "n_slices" in msg, (rc, msg)


def test_fast_rejects_a_launch_too_large_for_its_offsets(lib):
    """Maximum size: one fused launch holds fewer than 2^31 / 247 patients (the
    histogram drain forms 32-bit element offsets); a larger one is refused
    with GT_EINVAL before any CUDA call (no GPU needed), telling the caller to
    shard."""
    buf = C.create_string_buffer(64)
    a = _fast_args(n=9_000_000)
    for name, typ in a._fields_:
        if typ is C.c_void_p:
            setattr(a, name, C.addressof(buf))
        elif isinstance(typ, type) and issubclass(typ, C._Pointer):
            setattr(a, name, C.cast(C.addressof(buf), typ))
    rc, msg = _call_fast(lib, a)
    assert rc == -1 and "shard" in msg, (rc, msg)
