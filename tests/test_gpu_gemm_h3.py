"""The 3xF16 tensor-core GEMM (gemm_h3.cuh: power-of-two row/column operand
scales, hi/lo f16 split, kind::f16 MMAs) against a float64 reference with the
path's condition-aware tolerance |C - ref| <= 1e-5 * (|A| |B|), elementwise."""
import numpy as np
import pytest

from test_gpu_gemm import BIAS_TANH, NN, NT, STORE, TANH_GRAD, TN, dev, operands, run  # noqa: F401

pytestmark = pytest.mark.gpu

H3 = 4


@pytest.mark.parametrize("op", [NN, NT, TN])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 512, 2048), (192, 320, 96), (64, 4100, 36),
                                   (1024, 256, 256), (640, 384, 2048), (512, 128, 4096), (200, 260, 1000),
                                   # 80 pair tiles on 74 SM pairs: 74 whole tiles + 6 tiles as two
                                   # K halves each (tail-wave split, k_h3_tail_reduce); ragged edges
                                   (2560, 2048, 1024), (2500, 2020, 1000)])
def test_h3_store_condition_aware(dev, op, M, N, K):
    rs = np.random.default_rng(M * 7 + N * 3 + K + 1)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    out, _, launched = run(dev, op, M, N, K, A, B, STORE, use_tc=H3)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    err = np.abs(out - ref)
    assert launched in (3, 4)  # two operand-maxima passes + the kernel (+ the split-K / tail reduce)
    assert np.all(err <= 1e-5 * cond + 1e-30), f"max err/cond {np.max(err / (cond + 1e-30)):.3e}"


@pytest.mark.parametrize("op", [NN, NT, TN])
def test_h3_wide_dynamic_range(dev, op):
    # rows of op(A) and columns of op(B) spread over ~2^60 and individual
    # elements over another 2^20: the per-row / per-column scales keep every
    # output element within the condition-aware bound
    M, N, K = 256, 256, 512
    rs = np.random.default_rng(3 + op)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    ra = 2.0 ** rs.integers(-30, 30, M)
    cb = 2.0 ** rs.integers(-30, 30, N)
    ea = 2.0 ** rs.integers(-20, 1, (M, K))
    eb = 2.0 ** rs.integers(-20, 1, (K, N))
    Am = Am * ra[:, None] * ea
    Bm = Bm * cb[None, :] * eb
    Am = Am.astype(np.float32).astype(np.float64)
    Bm = Bm.astype(np.float32).astype(np.float64)
    A = np.ascontiguousarray((Am.T if op == TN else Am).astype(np.float32))
    B = np.ascontiguousarray((Bm.T if op == NT else Bm).astype(np.float32))
    out, _, _ = run(dev, op, M, N, K, A, B, STORE, use_tc=H3)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    err = np.abs(out - ref)
    assert np.all(err <= 1e-5 * cond + 1e-300), f"max err/cond {np.max(err / (cond + 1e-300)):.3e}"


def test_h3_zero_and_tiny_rows(dev):
    M, N, K = 128, 256, 256
    rs = np.random.default_rng(9)
    A, B, Am, Bm = operands(NN, M, N, K, rs)
    A[5] = 0.0
    A[7] *= 1e-30
    Am = A.astype(np.float64)
    out, _, _ = run(dev, NN, M, N, K, A, B, STORE, use_tc=H3)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    assert np.all(out[5] == 0.0)
    assert np.all(np.abs(out - ref) <= 1e-5 * cond + 1e-300)


@pytest.mark.parametrize("op", [NN, NT])
@pytest.mark.parametrize("M,N,K", [(256, 384, 512), (512, 256, 2048), (200, 260, 1000), (2560, 2048, 1024),
                                   # CTA pairs with ragged edges: the dgrad's TMA-prefetched
                                   # activations are clipped / zero-filled at M and N
                                   (2500, 2020, 1000), (4096, 2084, 2048)])
def test_h3_fused_epilogues(dev, op, M, N, K):
    rs = np.random.default_rng(5)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    A *= 0.1
    Am *= 0.1
    bias = rs.uniform(-0.5, 0.5, N).astype(np.float32)
    aux = rs.uniform(-0.99, 0.99, (M, N)).astype(np.float32)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    z, a, _ = run(dev, op, M, N, K, A, B, BIAS_TANH, bias=bias, use_tc=H3)
    assert np.all(np.abs(z - (ref + bias)) <= 1e-5 * cond + 1e-6)
    np.testing.assert_allclose(a, np.tanh(z.astype(np.float64)), rtol=2e-6, atol=2e-7)
    d, _, _ = run(dev, op, M, N, K, A, B, TANH_GRAD, aux=aux, use_tc=H3)
    g = (1 - aux.astype(np.float64) ** 2)
    assert np.all(np.abs(d - g * ref) <= 1e-5 * g * cond + 1e-6)


def test_h3_sass_uses_f16_tensor_cores(dev):
    import subprocess
    from paper_2001_04206_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    # kind::f16 MMAs show up as HMMA-class tcgen05 instructions in the k_gemm_h3 functions
    assert "k_gemm_h3" in sass


@pytest.mark.parametrize("op", [NN, NT, TN])
def test_h3_caller_maxima_bitwise(dev, op):
    # lane_b200_absmax + lane_b200_gemm_ex (the maxima the step computes once
    # per step) give the bits of the self-contained call
    import ctypes as C
    from paper_2001_04206_b200 import _native
    L = _native.lib()
    M, N, K = 1024, 512, 2048
    rs = np.random.default_rng(17 + op)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    ref, _, _ = run(dev, op, M, N, K, A, B, STORE, use_tc=H3)
    from test_gpu_gemm import put
    pa, pb = put(dev, A), put(dev, B)
    ar = (K, M) if op == TN else (M, K)
    br = (N, K) if op == NT else (K, N)
    bufs = [dev.alloc(4 * x) for x in (*ar, *br)]
    assert L.lane_b200_absmax(dev._p, C.c_void_p(pa), ar[0], ar[1], C.c_void_p(bufs[0]), C.c_void_p(bufs[1])) == 0
    assert L.lane_b200_absmax(dev._p, C.c_void_p(pb), br[0], br[1], C.c_void_p(bufs[2]), C.c_void_p(bufs[3])) == 0
    amax = bufs[1] if op == TN else bufs[0]
    bmax = bufs[2] if op == NT else bufs[3]
    pc = dev.alloc(M * N * 4)
    before = dev.kernel_launches
    rc = L.lane_b200_gemm_ex(dev._p, op, M, N, K, C.c_void_p(pa), C.c_void_p(pb), C.c_void_p(pc), None, None, None,
                             STORE, H3, C.c_void_p(amax), C.c_void_p(bmax))
    assert rc == 0, L.lane_b200_last_error()
    dev.sync()
    assert dev.kernel_launches - before in (1, 2)  # no maxima passes (+ the tail reduce)
    out = np.zeros((M, N), np.float32)
    dev.d2h(out, pc)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
    for p in (pa, pb, pc, *bufs):
        dev.free(p)
