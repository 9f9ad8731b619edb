"""Device-timed throughput of the mini-batch GEMMs (tcgen05 3xTF32 vs SIMT).

    python tools/bench_gemm.py
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [  # (name, op, M, N, K): the C3 step (B=256) and the C5 step (B=4096)
    ("c3.fwd1", 0, 256, 4096, 4096), ("c3.dgrad0", 1, 256, 4096, 4096), ("c3.wgrad1", 2, 4096, 4096, 256),
    ("c3.fwd0", 0, 256, 4096, 1024), ("c3.wgrad0", 2, 1024, 4096, 256),
    ("c5.fwd", 0, 4096, 4096, 4096), ("c5.dgrad", 1, 4096, 4096, 4096), ("c5.wgrad", 2, 4096, 4096, 4096),
]


def main():
    import torch
    from paper_2001_04206_b200 import _native, lane
    dev = lane.Device(0)
    L = _native.lib()
    stream = torch.cuda.ExternalStream(dev.stream)
    for name, op, M, N, K in SHAPES:
        a = torch.randn(M * K, device="cuda")
        b = torch.randn(N * K, device="cuda")
        c = torch.empty(M * N, device="cuda")
        for use_tc in [int(x) for x in os.environ.get("BENCH_TC", "1,0").split(",")]:
            def call():
                rc = L.lane_b200_gemm(dev._p, op, M, N, K, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                      C.c_void_p(c.data_ptr()), None, None, None, 0, use_tc)
                assert rc == 0, L.lane_b200_last_error()
            for _ in range(3):
                call()
            dev.sync()
            reps = 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                call()
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
            print(json.dumps({"gemm": name, "tc": use_tc, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                              "tflops_fp32_equiv": round(tf, 1)}), flush=True)


if __name__ == "__main__":
    main()
