"""CPU-side checks of the drop-in boundary: the C-ABI library builds for
sm_100a, loads, exports every symbol include/lane_b200.h declares, and fails
loudly (a status code + message, no crash, no CPU fallback) without a GPU."""
import ctypes as C
import os
import subprocess

import pytest
import torch

from paper_2001_04206_b200 import _build, _native


def test_library_exports_every_header_symbol():
    L = _native.load(check_gpu=False)
    declared = _native.header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/lane_b200.h but not exported"
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_native.SIGNATURES) == set(declared)
    assert L.lane_b200_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
    for other in ("sm_80", "sm_90", "sm_103"):
        assert other not in out.stdout


def test_kernels_present_in_sass():
    out = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    for k in ("k_sgd_cluster", "k_sgd_grid", "k_netin_strict", "k_delta_fc_strict", "k_outer",
              "k_apply_updates", "k_gemm_simt", "k_gemm_tc"):
        assert k in out, k


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_no_gpu_is_a_loud_error_not_a_fallback():
    L = _native.load(check_gpu=False)
    ctx = C.c_void_p()
    rc = L.lane_b200_ctx_create(0, C.byref(ctx))
    assert rc in (2, 7)  # ConfigError (no such device) or CUDA error
    assert L.lane_b200_last_error()
    from paper_2001_04206_b200 import lane
    with pytest.raises(lane.Error):
        lane.Device(0)


def test_library_then_torch_import_order():
    """liblane_b200.so links libnccl.so.2; loading it before torch must not
    bind the older system NCCL that torch's libtorch_cuda cannot use."""
    import subprocess
    import sys
    code = ("from paper_2001_04206_b200 import _native; _native.load(check_gpu=False); "
            "import torch; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
