"""The C boundary used from plain C (examples/c_api_demo.c, no CUDA headers):
compiled with gcc against include/fllf.h on CPU; run on the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_04681_b200", "lib")


def _build(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None or not os.path.exists(os.path.join(LIB, "libfllf.so")):
        pytest.skip("gcc or libfllf.so missing")
    exe = str(tmp_path / "c_api_demo")
    subprocess.run([gcc, "-O2", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", LIB, "-lfllf",
                    f"-Wl,-rpath,{LIB}", "-lm", "-o", exe], check=True)
    return exe


def test_c_api_demo_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_api_demo_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "c_api_demo ok" in r.stdout
