"""The boundary is a C ABI: a plain C program (examples/c_abi_demo.c, gcc, no Python in the
loop) creates a system, evaluates it on the device and checks the exact values, then runs
Alg. 2 to tolerance on x^2 - 4 from 1 (root 2 exactly)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_through_the_abi(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = str(tmp_path / "c_abi_demo")
    lib = os.path.join(ROOT, "paper_1109_0545_b200")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "c_abi_demo.c"), "-I" + os.path.join(ROOT, "include"),
                    "-L" + lib, "-lphc", "-I/usr/local/cuda/include", "-L/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "exact" in r.stdout
