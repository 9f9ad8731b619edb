"""The reference-side binding (integration/gpu_plan.hpp, INTEGRATION.md
section 2) at the reference's own call sites.

tests/native/test_gpu_plan.cpp is compiled against the REFERENCE's headers
and linked with the reference library built from its sources (oracle/Makefile
-> oracle/_ref/test_gpu_plan, where /root/reference exists; the binary
travels to the GPU box like oracle/_ref/liblane_ref.so).  On the GPU it runs
the reference's measure() loop (proj/src/bench.cpp:62-72) and train() with
lane::BackwardPlan and with lane::GpuPlan, STRICT numerics, and requires the
final hash_network and every LayerState buffer bit-identical.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "test_gpu_plan")
REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="compiles only where /root/reference exists")
def test_binding_compiles_against_reference_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_gpu_plan_measure_loop_and_train_bitwise_vs_reference():
    assert os.path.exists(EXE), "oracle/_ref/test_gpu_plan missing: run `make -C oracle` where /root/reference exists"
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu_plan ok" in r.stdout
