"""The C ABI from C: tests/c/abi_smoke.c includes include/liger_b200.h as C99, links
libliger_b200.so, and calls the host-only entry points (no GPU)."""

import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2410_10989_b200 import _capi

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_header_compiles_as_c_and_host_entry_points_answer(tmp_path):
    lib = Path(_capi.lib_path())
    _capi.load()  # builds the library if it is stale
    exe = tmp_path / "abi_smoke"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(ROOT / "tests" / "c" / "abi_smoke.c"),
           "-L", str(lib.parent), "-lliger_b200", f"-Wl,-rpath,{lib.parent}", "-o", str(exe)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "c abi ok" in run.stdout


@pytest.mark.gpu
@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_flce_through_the_c_abi_from_c(tmp_path):
    """tests/c/flce_c.c: cudaMalloc'd buffers, one lk_flce_forward_backward call (fp32), checked
    against a float64 loop restatement in C at the fp32 tolerance."""
    lib = Path(_capi.lib_path())
    _capi.load()
    cuda = Path("/usr/local/cuda")
    exe = tmp_path / "flce_c"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-I", str(cuda / "include"),
           str(ROOT / "tests" / "c" / "flce_c.c"), "-L", str(lib.parent), "-lliger_b200", f"-Wl,-rpath,{lib.parent}",
           "-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}", "-lm", "-o", str(exe)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "c flce ok" in run.stdout
