"""The C++ facade over the C ABI, compiled with g++ and run against the
in-tree liblane_b200.so (reference-style KATs in tests/native/test_facade.cpp)."""
import os
import subprocess

import pytest

from paper_2001_04206_b200 import _build

HERE = os.path.dirname(os.path.abspath(__file__))


def build_facade_test(tmp_path):
    exe = tmp_path / "test_facade"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(_build.ROOT, "include"),
                    os.path.join(HERE, "native", "test_facade.cpp"), "-o", str(exe),
                    "-L", _build.LIBDIR, "-llane_b200", f"-Wl,-rpath,{_build.LIBDIR}"], check=True)
    return exe


def test_facade_compiles_against_the_c_abi(tmp_path):
    _build.build()
    assert build_facade_test(tmp_path).exists()


@pytest.mark.gpu
def test_facade_reference_style_kats(tmp_path):
    _build.build()
    exe = build_facade_test(tmp_path)
    iris = os.path.join(HERE, "golden", "iris_normalized.txt")
    out = subprocess.run([str(exe), iris, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr
