"""3xF16 GEMM time against K at M = N = 4096 (lane_b200_gemm_ex with the
operand maxima precomputed, CUDA events, 10 reps): the slope per K is the
main loop, the intercept the fixed cost per GEMM.

    KS=512,1024,2048,4096,8192 python tools/gemm_kscan.py
    ZERO=1 KS=8192 REPS=200 python tools/gemm_kscan.py   # all-zero operands
"""
import ctypes as C
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_04206_b200 import _native, lane
dev = lane.Device(0); L = _native.lib()
stream = torch.cuda.ExternalStream(dev.stream)
M = N = 4096
for op, epi in ((0, 2), (1, 0), (2, 0)):
    for K in [int(k) for k in os.environ.get("KS", "512,1024,2048,4096,8192").split(",")]:
        ar = (K, M) if op == 2 else (M, K)
        br = (N, K) if op == 1 else (K, N)
        # ZERO=1: all-zero operands (the same work on data that toggles nothing)
        mk = torch.zeros if os.environ.get("ZERO") == "1" else torch.randn
        a = mk(ar, device="cuda"); b = mk(br, device="cuda")
        c = torch.empty(M * N, device="cuda"); c2 = torch.empty(M * N, device="cuda"); bias = torch.rand(N, device="cuda")
        bufs = [torch.zeros(x, dtype=torch.int32, device="cuda") for x in (*ar, *br)]
        torch.cuda.synchronize()
        assert L.lane_b200_absmax(dev._p, C.c_void_p(a.data_ptr()), ar[0], ar[1], C.c_void_p(bufs[0].data_ptr()), C.c_void_p(bufs[1].data_ptr())) == 0
        assert L.lane_b200_absmax(dev._p, C.c_void_p(b.data_ptr()), br[0], br[1], C.c_void_p(bufs[2].data_ptr()), C.c_void_p(bufs[3].data_ptr())) == 0
        amax = bufs[1] if op == 2 else bufs[0]; bmax = bufs[2] if op == 1 else bufs[3]
        def call():
            rc = L.lane_b200_gemm_ex(dev._p, op, M, N, K, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(c.data_ptr()),
                                     C.c_void_p(c2.data_ptr()), C.c_void_p(bias.data_ptr()), None, epi, 4,
                                     C.c_void_p(amax.data_ptr()), C.c_void_p(bmax.data_ptr()))
            assert rc == 0, L.lane_b200_last_error()
        for _ in range(3): call()
        dev.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = int(os.environ.get("REPS", "10"))
        for _ in range(reps): call()
        e1.record(stream); e1.synchronize()
        us = e0.elapsed_time(e1) * 1000 / reps
        print(json.dumps({"op": op, "epi": epi, "K": K, "us": round(us, 1), "tf": round(2.0 * M * N * K / us / 1e6, 1)}), flush=True)
