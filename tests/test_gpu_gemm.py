"""GEMMs of the mini-batch path (tcgen05 3xTF32 kernel and the SIMT kernel)
against a float64 numpy reference, with the condition-aware tolerance
|C - ref| <= 1e-5 * (|A| |B|)  elementwise."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NN, NT, TN = 0, 1, 2
STORE, BIAS, BIAS_TANH, TANH_GRAD = 0, 1, 2, 3


@pytest.fixture(scope="module")
def dev():
    from paper_2001_04206_b200 import lane
    d = lane.Device(0)
    yield d
    d.close()


def put(dev, a):
    a = np.ascontiguousarray(a, np.float32)
    p = dev.alloc(max(a.nbytes, 4))
    dev.h2d(p, a)
    return p


def run(dev, op, M, N, K, A, B, epi=STORE, bias=None, aux=None, use_tc=1):
    from paper_2001_04206_b200 import _native, lane
    L = _native.lib()
    pa, pb = put(dev, A), put(dev, B)
    pc, pc2 = dev.alloc(M * N * 4), dev.alloc(M * N * 4)
    pbias = put(dev, bias) if bias is not None else None
    paux = put(dev, aux) if aux is not None else None
    before = dev.kernel_launches
    rc = L.lane_b200_gemm(dev._p, op, M, N, K, C.c_void_p(pa), C.c_void_p(pb), C.c_void_p(pc),
                          C.c_void_p(pc2), C.c_void_p(pbias), C.c_void_p(paux), epi, use_tc)
    if rc:
        raise lane.Error(L.lane_b200_last_error().decode())
    dev.sync()
    out, out2 = np.zeros((M, N), np.float32), np.zeros((M, N), np.float32)
    dev.d2h(out, pc)
    dev.d2h(out2, pc2)
    for p in (pa, pb, pc, pc2, pbias, paux):
        if p:
            dev.free(p)
    return out, out2, dev.kernel_launches - before


def operands(op, M, N, K, rs):
    A = rs.uniform(-1, 1, (K, M) if op == TN else (M, K)).astype(np.float32)
    B = rs.uniform(-1, 1, (N, K) if op == NT else (K, N)).astype(np.float32)
    Am = A.T if op == TN else A
    Bm = B.T if op == NT else B
    return A, B, Am.astype(np.float64), Bm.astype(np.float64)


@pytest.mark.parametrize("use_tc", [1, 0, 2, 3])
@pytest.mark.parametrize("op", [NN, NT, TN])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 512, 2048), (256, 512, 1024), (192, 320, 96),
                                   (64, 4100, 36),
                                   (1024, 256, 256),
                                   # CTA-pair tiles (M >= 512, K >= 2048); 640 leaves the last
                                   # pair's second CTA entirely past M
                                   (640, 384, 2048), (512, 128, 4096)])
def test_gemm_store_condition_aware(dev, op, M, N, K, use_tc):
    rs = np.random.default_rng(M * 7 + N * 3 + K)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    out, _, launched = run(dev, op, M, N, K, A, B, STORE, use_tc=use_tc)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    err = np.abs(out - ref)
    # use_tc 2: the persistent kernel (stream-K pieces finished in-kernel);
    # 1 / 3: the one-tile-per-CTA kernel may split K (+1 fixed-order reduce)
    assert launched == 1 if use_tc in (0, 2) else launched in (1, 2)
    assert np.all(err <= 1e-5 * cond + 1e-30), f"max err/cond {np.max(err / (cond + 1e-30)):.3e}"


@pytest.mark.parametrize("use_tc", [1, 2])
@pytest.mark.parametrize("op", [NN, NT])
@pytest.mark.parametrize("M,N,K", [(256, 384, 512), (512, 256, 2048), (200, 260, 1000)])  # single, pairs, ragged
def test_gemm_fused_epilogues(dev, op, M, N, K, use_tc):
    rs = np.random.default_rng(5)
    A, B, Am, Bm = operands(op, M, N, K, rs)
    A *= 0.1
    Am *= 0.1
    bias = rs.uniform(-0.5, 0.5, N).astype(np.float32)
    aux = rs.uniform(-0.99, 0.99, (M, N)).astype(np.float32)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    z, a, _ = run(dev, op, M, N, K, A, B, BIAS_TANH, bias=bias, use_tc=use_tc)
    assert np.all(np.abs(z - (ref + bias)) <= 1e-5 * cond + 1e-6)
    np.testing.assert_allclose(a, np.tanh(z.astype(np.float64)), rtol=2e-6, atol=2e-7)
    d, _, _ = run(dev, op, M, N, K, A, B, TANH_GRAD, aux=aux, use_tc=use_tc)
    g = (1 - aux.astype(np.float64) ** 2)
    assert np.all(np.abs(d - g * ref) <= 1e-5 * g * cond + 1e-6)


def test_tensor_core_kernel_is_used(dev):
    # the eligible shape must run on the tcgen05 kernel, the ineligible one on SIMT
    import subprocess
    from paper_2001_04206_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    # A staged through TMEM (STTM) and the CTA-pair variant (2-CTA MMA + multicast commit)
    assert "STTM" in sass and "UTCHMMA.2CTA" in sass and "UTCBAR.2CTA.MULTICAST" in sass


@pytest.mark.parametrize("epi", [STORE, TANH_GRAD])
def test_shortk_nt_output_layer_dgrad(dev, epi):
    # D[M][K<=16] W[N][K]^T (x tanh'), the 10-class output layer's dgrad
    M, N, K = 256, 4100, 10
    rs = np.random.default_rng(11)
    A, B, Am, Bm = operands(NT, M, N, K, rs)
    aux = rs.uniform(-0.99, 0.99, (M, N)).astype(np.float32)
    out, _, launched = run(dev, NT, M, N, K, A, B, epi, aux=aux if epi == TANH_GRAD else None)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    g = (1 - aux.astype(np.float64) ** 2) if epi == TANH_GRAD else 1.0
    assert launched == 1
    assert np.all(np.abs(out - g * ref) <= 1e-5 * g * cond + 1e-30)


@pytest.mark.parametrize("M,N,K", [(4096, 10, 4096), (1024, 16, 1000), (520, 3, 2049), (4100, 10, 700),
                                   (256, 10, 4096)])
def test_skinny_tn_long_k(dev, M, N, K):
    # op(A)^T B with N <= 16 and a long K: the output layer's wgrad
    rs = np.random.default_rng(13)
    A, B, Am, Bm = operands(TN, M, N, K, rs)
    out, _, launched = run(dev, TN, M, N, K, A, B, STORE)
    ref = Am @ Bm
    cond = np.abs(Am) @ np.abs(Bm)
    assert launched == 2
    assert np.all(np.abs(out - ref) <= 1e-5 * cond + 1e-30)


@pytest.mark.parametrize("epi", [STORE, BIAS, BIAS_TANH])
@pytest.mark.parametrize("M,N,K", [(256, 10, 4096 + 96), (4096, 10, 4096), (2100, 16, 2048), (3000, 3, 1100),
                                   (256, 10, 2050)])
def test_skinny_nn_long_k(dev, epi, M, N, K):
    # A[M][K] B[K][N<=16] with a long K: chunked, fixed-order partial sums
    # (row per lane for M >= 2048 and K % 4 == 0, incl. C5's output layer; lanes along K otherwise)
    rs = np.random.default_rng(12)
    A, B, Am, Bm = operands(NN, M, N, K, rs)
    A *= 0.05
    Am *= 0.05
    bias = rs.uniform(-0.5, 0.5, N).astype(np.float32)
    out, out2, launched = run(dev, NN, M, N, K, A, B, epi, bias=bias if epi != STORE else None)
    ref = Am @ Bm + (bias if epi != STORE else 0.0)
    cond = np.abs(Am) @ np.abs(Bm)
    assert launched == 2
    assert np.all(np.abs(out - ref) <= 1e-5 * cond + 1e-6)
    if epi == BIAS_TANH:
        np.testing.assert_allclose(out2, np.tanh(out.astype(np.float64)), rtol=2e-6, atol=2e-7)
