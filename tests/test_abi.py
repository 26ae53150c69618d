"""Host-side checks of the C-ABI library that need no GPU: it builds for sm_100a, loads, exports
every entry point declared in include/bn.h, and fails loudly (never falls back) without a device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bn.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_2105_12620_b200 import build

    return build.build()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bn_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    # lattice/generator setup, bank setup, error-vector evaluation, energy, optimise, readback
    for need in ("bn_set_lattice", "bn_set_bank", "bn_eval_counts", "bn_energy", "bn_optimize", "bn_get_tile"):
        assert need in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bn_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_binding_lists_every_symbol():
    from paper_2105_12620_b200 import bn

    assert sorted(bn.SYMBOLS) == declared_symbols()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string(libpath):
    from paper_2105_12620_b200 import bn

    assert "sm_100a" in bn.version()


def test_no_device_fails_loudly(libpath):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2105_12620_b200 import bn

    lib = bn.load_library()
    ctx = ctypes.c_void_p()
    assert lib.bn_create(ctypes.byref(ctx), 0, 0) == bn.BN_ECUDA
    assert not ctx.value


def test_null_context_is_einval(libpath):
    from paper_2105_12620_b200 import bn

    lib = bn.load_library()
    lv = (ctypes.c_uint32 * 1)(16)
    assert lib.bn_set_lattice(None, 1, 27, lv, 1) == bn.BN_EINVAL
    assert lib.bn_set_energy(None, 2.1, 1.0, 7) == bn.BN_EINVAL
    assert lib.bn_launch_count(None) == 0


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2105_12620_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("no CPU fallback", ""), f
