"""Loader for liblane_b200.so (the C ABI in include/lane_b200.h).

No fallback: if the library is missing it is built with nvcc (sm_100a), and
if that fails the import error propagates.  ``load(check_gpu=False)`` only
loads the library (used by the CPU test that checks the exported symbols).
"""
from __future__ import annotations

import ctypes as C
import os
import re

from . import _build

_lib = None

_V = C.c_void_p
_S = C.c_size_t
_I = C.c_int
_F = C.c_float
_FP = C.POINTER(C.c_float)
_SP = C.POINTER(C.c_size_t)
_U64 = C.c_uint64

SIGNATURES = {
    "lane_b200_abi_version": (_I, []),
    "lane_b200_last_error": (C.c_char_p, []),
    "lane_b200_ctx_create": (_I, [_I, C.POINTER(_V)]),
    "lane_b200_ctx_destroy": (_I, [_V]),
    "lane_b200_ctx_set_numerics": (_I, [_V, _I]),
    "lane_b200_ctx_get_numerics": (_I, [_V, C.POINTER(_I)]),
    "lane_b200_sync": (_I, [_V]),
    "lane_b200_ctx_stream": (_I, [_V, C.POINTER(_V)]),
    "lane_b200_kernel_launches": (_I, [_V, C.POINTER(_U64)]),
    "lane_b200_dev_alloc": (_I, [_V, _S, C.POINTER(_V)]),
    "lane_b200_dev_free": (_I, [_V, _V]),
    "lane_b200_memcpy_h2d": (_I, [_V, _V, _V, _S]),
    "lane_b200_memcpy_d2h": (_I, [_V, _V, _V, _S]),
    "lane_b200_net_create": (_I, [_V, _S, _SP, _S, _S, _S, C.POINTER(_V)]),
    "lane_b200_net_init_seeded": (_I, [_V, _U64]),
    "lane_b200_net_destroy": (_I, [_V]),
    "lane_b200_net_shape": (_I, [_V, _S, _SP, _SP]),
    "lane_b200_net_n_layers": (_I, [_V, _SP]),
    "lane_b200_buf_read": (_I, [_V, _S, _I, _FP, _S]),
    "lane_b200_buf_write": (_I, [_V, _S, _I, _FP, _S]),
    "lane_b200_buf_device_ptr": (_I, [_V, _S, _I, C.POINTER(_FP), _SP]),
    "lane_b200_net_hash": (_I, [_V, C.POINTER(_U64)]),
    "lane_b200_layer_forward": (_I, [_V, _S, _FP, _S]),
    "lane_b200_fc_backward": (_I, [_V, _S, _FP, _S, _S, _FP, _S, _F]),
    "lane_b200_softmax_backward": (_I, [_V, _FP, _S, _F]),
    "lane_b200_apply_updates": (_I, [_V, _S]),
    "lane_b200_forward": (_I, [_V, _FP, _FP]),
    "lane_b200_backward_plan_run": (_I, [_V, _FP, _F]),
    "lane_b200_backward_plan_run_timed": (_I, [_V, _FP, _F, C.POINTER(C.c_double), _S]),
    "lane_b200_sgd_stream": (_I, [_V, _V, _V, _S, _V, _S, _F, _V, _V]),
    "lane_b200_sgd_stream_plan": (_I, [_V, C.c_char_p, _S]),
    "lane_b200_train": (_I, [_V, _FP, _FP, _S, _F, _F, _S, _U64, _FP, _FP, _SP]),
    "lane_b200_evaluate": (_I, [_V, _FP, _FP, _S, _FP, _FP]),
    "lane_b200_minibatch_step": (_I, [_V, _V, _V, _S, _F, _F, _V]),
    "lane_b200_minibatch_grads": (_I, [_V, _V, _V, _S, _V]),
    "lane_b200_minibatch_apply": (_I, [_V, _S, _F, _F]),
    "lane_b200_net_grads_arena": (_I, [_V, _V, _V]),
    "lane_b200_train_minibatch": (_I, [_V, _FP, _FP, _S, _S, _F, _F, _S, _U64, _I, _I, _FP, _FP, _SP]),
    "lane_b200_dataset_create": (_I, [_S, _S, _S, _FP, _FP, C.POINTER(_V)]),
    "lane_b200_dataset_load": (_I, [C.c_char_p, _S, _S, C.POINTER(_V)]),
    "lane_b200_dataset_save": (_I, [_V, C.c_char_p]),
    "lane_b200_dataset_info": (_I, [_V, _SP, _SP, _SP, C.POINTER(_FP), C.POINTER(_FP), C.POINTER(_I)]),
    "lane_b200_dataset_split": (_I, [_V, C.c_double, _U64, C.POINTER(_V), C.POINTER(_V)]),
    "lane_b200_dataset_enlarge": (_I, [_V, _S, _F, C.POINTER(_U64), C.POINTER(_V)]),
    "lane_b200_dataset_destroy": (_I, [_V]),
    "lane_b200_gemm": (_I, [_V, _I, _I, _I, _I, _V, _V, _V, _V, _V, _V, _I, _I]),
    "lane_b200_gemm_ex": (_I, [_V, _I, _I, _I, _I, _V, _V, _V, _V, _V, _V, _I, _I, _V, _V]),
    "lane_b200_absmax": (_I, [_V, _V, _I, _I, _V, _V]),
    "lane_b200_nccl_unique_id": (_I, [_V, _S]),
    "lane_b200_comm_init": (_I, [_V, _I, _I, _V, _S]),
    "lane_b200_comm_destroy": (_I, [_V]),
    "lane_b200_allreduce_grads": (_I, [_V]),
    "lane_b200_nvls_supported": (_I, [_V, C.POINTER(_I)]),
    "lane_b200_nvls_create": (_I, [_V, _I, C.POINTER(_I)]),
    "lane_b200_nvls_attach": (_I, [_V, _I, _I, _I]),
    "lane_b200_nvls_bind": (_I, [_V]),
    "lane_b200_nvls_mode": (_I, [_V, C.POINTER(_I)]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/lane_b200.h."""
    hdr = os.path.join(_build.ROOT, "include", "lane_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(lane_b200_[a-z0-9_]+)\s*\(", text)))


def _preload_torch_nccl() -> None:
    """PyTorch ships its own libnccl.so.2, newer than the system one that
    liblane_b200.so is linked against.  Both are found by the soname
    libnccl.so.2, and the first one loaded wins.  If the system copy came
    first, a later ``import torch`` would fail on missing NCCL symbols. So the
    bundled copy (a superset of the API this library calls) is loaded globally
    before this library, and torch and the library share one NCCL whichever is
    imported first."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for base in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(p):
            C.CDLL(p, mode=C.RTLD_GLOBAL)
            return


def load(check_gpu: bool = True):
    global _lib
    if _lib is None:
        # LANE_B200_LIB: an alternative build of the same library (experiments)
        path = os.environ.get("LANE_B200_LIB") or _build.build()  # no-op when up to date
        _preload_torch_nccl()
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def lib():
    return load()
