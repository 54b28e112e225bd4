"""Builds tests/cpp/test_api.cpp against include/ctsm_b200/ctsm.hpp and
libctsm_b200.so (the C++ drop-in) and runs it on the GPU."""
import os
import subprocess

import pytest

from paper_2511_12235_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api_compiles(tmp_path):
    exe = tmp_path / "test_api"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), _lib.LIB_PATH,
                    "-Wl,-rpath," + os.path.dirname(_lib.LIB_PATH), "-ldl", "-pthread", "-o", str(exe)],
                   check=True)
    assert exe.exists()


@pytest.mark.gpu
def test_cpp_api_on_gpu(tmp_path):
    exe = tmp_path / "test_api"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), _lib.LIB_PATH,
                    "-Wl,-rpath," + os.path.dirname(_lib.LIB_PATH), "-ldl", "-pthread", "-o", str(exe)],
                   check=True)
    env = dict(os.environ)
    ref = os.path.join(ROOT, "oracle", "_ref", "libctsm_ref_cr.so")
    if os.path.exists(ref):  # the unmodified reference with the correctly rounded libm
        env["CTSM_TEST_ORACLE_LIB"] = ref
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
