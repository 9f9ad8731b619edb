"""The device transcendental functions (paper_2001_04206_b200/csrc/lane_libm.cuh)
restate glibc's tanhf/expf/logf.  Their host build is compared against the
running glibc over a strided sweep of ALL 2^32 float bit patterns (stride 1,
i.e. exhaustive, when LANE_FULL_LIBM=1; ~27 s on 8 cores).  The device build
uses the same code with never-contracted __*_rn intrinsics; the GPU test
tests/test_gpu_parity.py::test_device_tanhf_bitwise_vs_glibc closes the loop."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_libm_restatement_matches_glibc(tmp_path):
    exe = tmp_path / "libm_ex"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-o", str(exe),
                    os.path.join(HERE, "native", "libm_exhaustive.cpp"), "-lm"], check=True)
    stride = "1" if os.environ.get("LANE_FULL_LIBM") == "1" else "61"
    out = subprocess.run([str(exe), stride], capture_output=True, text=True)
    assert "TOTAL_MISMATCHES 0" in out.stdout, out.stdout
    assert out.returncode == 0
