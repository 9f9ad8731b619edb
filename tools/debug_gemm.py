"""Structured-input probes of the tcgen05 GEMM (layout debugging)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2001_04206_b200 import _native, lane
    dev = lane.Device(0)
    L = _native.lib()
    M = N = 128
    K = 32
    res = {}

    def run(op, A, B):
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        pa, pb, pc = dev.alloc(A.nbytes), dev.alloc(B.nbytes), dev.alloc(M * N * 4)
        dev.h2d(pa, A)
        dev.h2d(pb, B)
        rc = L.lane_b200_gemm(dev._p, op, M, N, K, C.c_void_p(pa), C.c_void_p(pb), C.c_void_p(pc), None, None,
                              None, 0, 1)
        assert rc == 0, L.lane_b200_last_error()
        dev.sync()
        out = np.zeros((M, N), np.float32)
        dev.d2h(out, pc)
        for p in (pa, pb, pc):
            dev.free(p)
        return out

    # encode positions: A[m][k] = m + k/100 style codes with one-hot partner
    for op in (0, 1, 2):
        # probe 1: A one-hot picks B rows (C[m][n] = B(k=m%K, n) for m < K)
        Am = np.zeros((M, K), np.float32)
        for m in range(K):
            Am[m, m] = 1
        Bm = (np.arange(K)[:, None] * 1000 + np.arange(N)[None, :]).astype(np.float32)  # B(k, n) = 1000k + n
        A = Am.T if op == 2 else Am
        B = Bm.T if op == 1 else Bm
        res[f"p1_op{op}"] = run(op, A, B)
        # probe 2: B one-hot picks A columns (C[m][n] = A(m, k=n) for n < K)
        Bm2 = np.zeros((K, N), np.float32)
        for k in range(K):
            Bm2[k, k] = 1
        Am2 = (np.arange(M)[:, None] * 1000 + np.arange(K)[None, :]).astype(np.float32)  # A(m, k) = 1000m + k
        A = Am2.T if op == 2 else Am2
        B = Bm2.T if op == 1 else Bm2
        res[f"p2_op{op}"] = run(op, A, B)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez("gpurun_out/debug_gemm.npz", **res)
    print("saved")


if __name__ == "__main__":
    main()
