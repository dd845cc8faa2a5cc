"""The C++ drop-in (include/chebstep/*.hpp, namespace chebstep) called the way the
reference's own callers call it, checked against the compiled reference library."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "dropin_test")


def build_dropin():
    lib = os.path.join(ROOT, "paper_2603_09790_b200", "lib")
    ref = os.path.join(ROOT, "oracle", "_ref")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"),
           "-o", EXE, "-L", lib, "-lchebstep_gpu", "-L", ref, "-lchebstep_ref",
           f"-Wl,-rpath,{lib}:{ref}"]
    import glob
    ob = glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/opencv_python_headless.libs")
    if ob:
        cmd.append(f"-Wl,-rpath-link,{ob[0]}")
    subprocess.run(cmd, check=True)


def test_cpp_dropin():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libchebstep_ref.so")):
        pytest.skip("reference oracle not built")
    build_dropin()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "DROPIN OK" in out.stdout, out.stdout + out.stderr
