"""The boundary from plain C99: compile tests/c_abi_check.c against include/mlfabric.h and
link it to libmlfabric.so with gcc, then run it (host-only planner calls; no GPU)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(ROOT, "paper_1907_00434_b200", "lib")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_c99_program_against_the_abi(tmp_path):
    exe = tmp_path / "c_abi_check"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(HERE, "c_abi_check.c"), "-o", str(exe), "-L", LIB, "-lmlfabric",
                    f"-Wl,-rpath,{LIB}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "C_ABI_OK" in r.stdout, r.stdout + r.stderr
