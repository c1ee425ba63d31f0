"""CPU-side checks of the C-ABI boundary: libasim.so builds for sm_100a,
loads without a GPU, and exports every entry point include/asim.h declares;
the Python binding raises (no fallback) when no device is present."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            src = open(os.path.join(ROOT, "include", f)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(asim_[a-z_]+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def libpath():
    from paper_2302_11665_b200 import build
    return build.build()


def test_header_declares_entry_points():
    names = _declared()
    for n in ["asim_create", "asim_destroy", "asim_set_problem", "asim_set_trace",
              "asim_evaluate", "asim_evaluate_deltas", "asim_attainment", "asim_search_create",
              "asim_search_prepare", "asim_search_evaluate", "asim_search_apply"]:
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = _declared() - exported
    assert not missing, missing


def test_library_is_sm100a(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                                  text=True)
    assert "sm_100a" in out


def test_binding_loads_and_names_match(libpath):
    from paper_2302_11665_b200 import _abi
    assert _abi.asim_abi_version() == 1
    assert set(_abi.EXPORTED) >= _declared()
    assert _abi.asim_attainment(3, 4) == 0.75
    assert _abi.asim_attainment(0, 0) == 1.0
    assert _abi.asim_attainment(-1, 5) == -1.0


def test_create_without_gpu_fails_loudly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2302_11665_b200 import AsimError, Simulator
    with pytest.raises(AsimError):
        Simulator(0)
