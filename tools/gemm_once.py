"""Run one GEMM shape a few times through lane_b200_gemm (for ncu captures).

    python tools/gemm_once.py OP M N K USE_TC [EPI] [REPS]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2001_04206_b200 import _native, lane
    op, M, N, K, use_tc = (int(x) for x in sys.argv[1:6])
    epi = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
    dev = lane.Device(0)
    L = _native.lib()
    a = torch.rand(M * K, device="cuda") - 0.5
    b = torch.rand(N * K, device="cuda") - 0.5
    c = torch.empty(M * N, device="cuda")
    c2 = torch.empty(M * N, device="cuda")
    bias = torch.rand(N, device="cuda")
    aux = torch.rand(M * N, device="cuda")
    torch.cuda.synchronize()
    for _ in range(reps):
        rc = L.lane_b200_gemm(dev._p, op, M, N, K, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                              C.c_void_p(c.data_ptr()), C.c_void_p(c2.data_ptr()), C.c_void_p(bias.data_ptr()),
                              C.c_void_p(aux.data_ptr()), epi, use_tc)
        assert rc == 0, L.lane_b200_last_error()
    dev.sync()


if __name__ == "__main__":
    main()
