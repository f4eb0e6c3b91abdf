"""The C ABI used from C (no Python in the loop): tests/c_abi/heat_host.c
compiles against include/tilemesh_b200.h here (CPU) and runs on the GPU:
FillBoundary as copy tags, three heat sweeps and the checksum, bit-exact
against its own C restatement of the reference arithmetic."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SRC = os.path.join(ROOT, "tests", "c_abi", "heat_host.c")
LIBDIR = os.path.join(ROOT, "paper_1604_03570_b200")


def compile_host(out, link=True):
    cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC]
    if link:
        cmd += ["-o", out, "-L", LIBDIR, "-ltilemesh_b200", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    else:
        cmd += ["-c", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not found")
def test_c_host_compiles_against_header(tmp_path):
    compile_host(str(tmp_path / "heat_host.o"), link=False)


@pytest.mark.gpu
def test_c_host_runs_bit_exact(tmp_path):
    exe = str(tmp_path / "heat_host")
    compile_host(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "c-abi ok" in r.stdout
