"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

The oracle (oracle/lane_oracle.c) is pinned bit-for-bit to the reference by
tests/test_oracle.py; the golden fixture tests/golden/golden.npz comes from
the reference itself.

Tolerances:
  STRICT numerics: bit-identical -- every buffer, every step, every epoch
    statistic (the device uses the reference's evaluation order, separately
    rounded mul/add, and bit-exact restatements of glibc tanhf/expf/logf).
  FAST numerics: per step, every reduced quantity within
    |gpu - cpu| <= 1e-5 * sum_k |a_k * b_k| (condition-aware), checked here in
    its normwise form max|gpu - cpu| <= 1e-5 * max|cpu| per buffer;
    over an epoch, mean loss within 1e-4 relative and identical accuracy
    counts up to argmax ties.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
IRIS = os.path.join(os.path.dirname(__file__), "golden", "iris_normalized.txt")
BUFS = ("weights", "gradients", "delta_weights", "biases", "inputs", "netin", "outputs",
        "deltas", "delta_biases")


@pytest.fixture(scope="module")
def lane():
    from paper_2001_04206_b200 import lane as L
    return L


@pytest.fixture(scope="module")
def dev(lane):
    d = lane.Device(0)
    yield d
    d.close()


@pytest.fixture
def strict(dev, lane):
    old = dev.numerics
    dev.numerics = lane.NUMERICS_STRICT
    yield dev
    dev.numerics = old


@pytest.fixture
def fast(dev, lane):
    old = dev.numerics
    dev.numerics = lane.NUMERICS_FAST
    yield dev
    dev.numerics = old


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(a, b, what=""):
    a, b = np.asarray(a, np.float32).reshape(-1), np.asarray(b, np.float32).reshape(-1)
    bad = np.nonzero(bits(a) != bits(b))[0]
    assert bad.size == 0, f"{what}: {bad.size} of {a.size} differ, first {bad[:5]} " \
                          f"gpu {a[bad[:5]]} cpu {b[bad[:5]]}"


def assert_close(gpu, cpu, rtol=1e-5, what=""):
    gpu, cpu = np.asarray(gpu, np.float64).reshape(-1), np.asarray(cpu, np.float64).reshape(-1)
    scale = max(np.max(np.abs(cpu)), 1e-30)
    err = np.max(np.abs(gpu - cpu)) if cpu.size else 0.0
    assert err <= rtol * scale, f"{what}: normwise err {err / scale:.3e} > {rtol:g}"


def layer_arrays(layer):
    return {b: getattr(layer, b) for b in BUFS}


def oracle_arrays(orc, l):
    return {b: orc.get(l, i) for i, b in enumerate(BUFS)}


# ------------------------------------------------------------ init ----------

@pytest.mark.parametrize("F,H,C", [(4, [8], 3), (784, [128], 10), (16, [12, 9], 5), (3, [], 2)])
def test_build_network_bitwise(lane, dev, F, H, C):
    net = lane.build_network(F, H, C, seed=42, device=dev)
    orc = po.OracleNet(F, H, C, seed=42)
    for l, layer in enumerate(net.layers):
        assert_bitwise(layer.weights, orc.get(l, po.W), f"W{l}")
        assert not np.any(layer.biases)
    assert net.hash() == orc.hash()


def test_device_tanhf_bitwise_vs_glibc(lane, strict):
    # Layer with I=1, W[0][j] = z_j, x = 1: netin_j = (0 + 1*z_j) + 0 = z_j, a = tanhf(z_j)
    rs = np.random.default_rng(3)
    z = np.concatenate([rs.standard_normal(40000) * 4, rs.uniform(-30, 30, 20000),
                        rs.standard_normal(4000) * 1e-3,
                        np.float32([0.0, 1.0, -1.0, 22.0, 9.01, 0.5493, -0.3466])]).astype(np.float32)
    net = lane.FeedForwardNetwork(1, [z.size], 2, device=strict)
    net.hidden[0].weights = z.reshape(1, -1)
    a = net.hidden[0].forward(np.ones(1, np.float32))
    libm = C.CDLL("libm.so.6")
    libm.tanhf.restype, libm.tanhf.argtypes = C.c_float, [C.c_float]
    want = np.array([libm.tanhf(float(v)) for v in z], np.float32)
    assert_bitwise(net.hidden[0].netin, z, "netin")
    assert_bitwise(a, want, "tanhf")


# ------------------------------------------------------- layer KATs ---------

def test_softmax_backward_hand_kat(lane, dev):
    # proj/tests/test_layers.cpp:125-142 (layer 1 -> 2 as the output of a 1-[1]-2 net)
    net = lane.FeedForwardNetwork(3, [1], 2, device=dev)
    out = net.output
    out.outputs = [0.7, 0.3]
    out.inputs = [2.0]
    out.backward([1.0, 0.0], lane.LearningRate(0.1))
    np.testing.assert_allclose(out.deltas, [-0.3, 0.3], rtol=1e-6)
    np.testing.assert_allclose(out.gradients[0], [-0.6, 0.6], rtol=1e-6)
    np.testing.assert_allclose(out.delta_weights[0], [0.06, -0.06], rtol=1e-6)
    np.testing.assert_allclose(out.delta_biases, [0.03, -0.03], rtol=1e-6)
    with pytest.raises(lane.ShapeError):
        out.backward([1.0], lane.LearningRate(0.1))


def test_fc_backward_hand_kat_and_shape_errors(lane, dev):
    # proj/tests/test_layers.cpp:209-222
    net = lane.FeedForwardNetwork(1, [1], 2, device=dev)
    h = net.hidden[0]
    h.outputs = [0.5]
    h.inputs = [1.0]
    h.backward(np.array([[3.0]]), [0.2], lane.LearningRate(0.1))
    np.testing.assert_allclose(h.deltas, [0.45], rtol=1e-6)
    with pytest.raises(lane.ShapeError):
        h.backward(np.zeros((2, 1)), [0.2], lane.LearningRate(0.1))
    with pytest.raises(lane.ShapeError):
        h.backward(np.zeros((1, 1)), [0.2, 0.3], lane.LearningRate(0.1))


def test_zero_signal_cases(lane, dev):
    # proj/tests/test_layers.cpp:144-161, :224-238
    net = lane.FeedForwardNetwork(2, [3], 3, device=dev)
    net.output.outputs = [0, 1, 0]
    net.output.inputs = [0.4, -0.2, 0.1]
    net.output.backward([0, 1, 0], 0.5)
    for b in ("deltas", "gradients", "delta_weights", "delta_biases"):
        assert not np.any(getattr(net.output, b))
    net.hidden[0].forward([0.5, -0.5])
    net.hidden[0].backward(np.ones((3, 2)), [0.0, 0.0], 0.1)
    assert not np.any(net.hidden[0].deltas) and not np.any(net.hidden[0].gradients)


def test_apply_updates_kat(lane, dev):
    # proj/tests/test_layers.cpp:240-258
    net = lane.FeedForwardNetwork(1, [1], 2, device=dev)
    h = net.hidden[0]
    h.weights = [[1.0]]
    h.delta_weights = [[-0.06]]
    h.delta_biases = [0.5]
    h.apply_updates()
    assert h.weights[0, 0] == np.float32(0.94) and h.biases[0] == np.float32(0.5)
    h.apply_updates()
    np.testing.assert_allclose(h.weights[0, 0], 0.88, rtol=1e-6)


def test_learning_rate_must_be_positive(lane, dev):
    with pytest.raises(lane.ConfigError):
        lane.LearningRate(0.0)
    net = lane.FeedForwardNetwork(2, [2], 2, device=dev)
    with pytest.raises(lane.ConfigError):
        net.output.backward([1, 0], -0.1)
    with pytest.raises(lane.ConfigError):
        lane.FeedForwardNetwork(2, [0], 2, device=dev)
    with pytest.raises(lane.ConfigError):
        lane.FeedForwardNetwork(2, [3], 1, device=dev)


# --------------------------------------- layer backward / forward vs golden -

@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_layer_backward_matches_reference_golden(lane, dev, mode):
    dev.numerics = lane.NUMERICS_STRICT if mode == "strict" else lane.NUMERICS_FAST
    try:
        for c in range(24):
            I, O = GOLD[f"smb{c}_shape"]
            v = GOLD[f"smb{c}_in"]
            net = lane.FeedForwardNetwork(3, [I], O, device=dev)
            net.output.outputs = v[:O]
            net.output.inputs = v[O:O + I]
            net.output.backward(v[O + I:], 0.05)
            for k in ("deltas", "gradients", "delta_weights", "delta_biases"):
                assert_bitwise(getattr(net.output, k), GOLD[f"smb{c}_{k}"], f"smb{c} {k}")
        for c in range(24):
            I, O, N = GOLD[f"fcb{c}_shape"]
            v = GOLD[f"fcb{c}_in"]
            net = lane.FeedForwardNetwork(I, [O], 2, device=dev)
            h = net.hidden[0]
            h.outputs = v[:O]
            h.inputs = v[O:O + I]
            h.backward(v[O + I:O + I + O * N].reshape(O, N), v[O + I + O * N:], 0.05)
            for k in ("deltas", "gradients", "delta_weights", "delta_biases"):
                assert_bitwise(getattr(h, k), GOLD[f"fcb{c}_{k}"], f"fcb{c} {k}")
    finally:
        dev.numerics = lane.NUMERICS_FAST


def test_layer_forward_matches_reference_golden_strict(lane, strict):
    for c in range(16):
        W, b, x = GOLD[f"fwd{c}_W"], GOLD[f"fwd{c}_b"], GOLD[f"fwd{c}_x"]
        I, O = W.shape
        if c % 2:  # softmax layer = output of a (I)-[]-(O) net
            net = lane.FeedForwardNetwork(I, [], O, device=strict)
            layer = net.output
        else:
            net = lane.FeedForwardNetwork(I, [O], 2, device=strict)
            layer = net.hidden[0]
        layer.weights = W
        layer.biases = b
        layer.forward(x)
        assert_bitwise(layer.netin, GOLD[f"fwd{c}_z"], f"fwd{c} z")
        assert_bitwise(layer.outputs, GOLD[f"fwd{c}_a"], f"fwd{c} a")


@pytest.mark.parametrize("I,O", [(340, 4096), (4096, 10), (784, 128), (1024, 257)])
def test_layer_forward_fast_within_tolerance(lane, fast, I, O):
    rs = np.random.default_rng(I + O)
    W = (rs.uniform(-1, 1, (I, O)) / np.sqrt(I)).astype(np.float32)
    b = rs.uniform(-0.1, 0.1, O).astype(np.float32)
    x = rs.uniform(0, 1, I).astype(np.float32)
    net = lane.FeedForwardNetwork(I, [O], 2, device=fast)
    net.hidden[0].weights = W
    net.hidden[0].biases = b
    net.hidden[0].forward(x)
    z_ref, a_ref = po.oracle_layer_forward("fc", W, b, x)
    cond = np.abs(x)[:, None].T @ np.abs(W)  # sum_i |x_i W_ij|
    err = np.abs(net.hidden[0].netin.astype(np.float64) - z_ref)
    assert np.all(err <= 1e-5 * cond.reshape(-1) + 1e-30)
    assert_close(net.hidden[0].outputs, a_ref, 1e-5, "a")


# ---------------------------------------------------- network steps ---------

@pytest.mark.parametrize("name,F,H,C,eta,steps", [
    ("c1", 4, [8], 3, 0.01, 4), ("c2", 784, [128], 10, 0.01, 3),
    ("c4", 340, [256], 10, 1e-4, 2), ("deep", 16, [12, 9], 5, 0.05, 4)])
def test_backward_plan_steps_bitwise_vs_reference_golden(lane, strict, name, F, H, C, eta, steps):
    X, T = po.synthetic_dataset(F, C, 8, 9)
    net = lane.build_network(F, H, C, seed=42, device=strict)
    plan = lane.BackwardPlan(net, lane.LearningRate(eta))
    assert net.hash() == int(GOLD[f"{name}_hash0"][0])
    for s in range(steps):
        assert_bitwise(net.forward(X[s]), GOLD[f"{name}_probs"][s], f"probs step {s}")
        plan.run(T[s])
        assert net.hash() == int(GOLD[f"{name}_hashes"][s]), f"weights hash step {s}"
        d = np.concatenate([layer.deltas for layer in net.layers])
        assert_bitwise(d, GOLD[f"{name}_deltas"][s], f"deltas step {s}")


def test_backward_plan_all_buffers_bitwise_vs_oracle(lane, strict):
    X, T = po.synthetic_dataset(50, 7, 4, 1)
    net = lane.build_network(50, [33, 17], 7, seed=5, device=strict)
    orc = po.OracleNet(50, [33, 17], 7, seed=5)
    for s in range(4):
        net.forward(X[s])
        orc.forward(X[s])
        lane.BackwardPlan(net, 0.02).run(T[s])
        orc.backward_plan_run(T[s], 0.02)
        for l, layer in enumerate(net.layers):
            got, want = layer_arrays(layer), oracle_arrays(orc, l)
            for b in BUFS:
                assert_bitwise(got[b], want[b], f"step {s} layer {l} {b}")


# ------------------------------------------ fused persistent online SGD -----

def upload(dev, a, dtype=np.float32):
    a = np.ascontiguousarray(a, dtype)
    p = dev.alloc(a.nbytes)
    dev.h2d(p, a)
    return p


@pytest.mark.parametrize("F,H,C,n,steps,eta,ctas", [
    (784, [128], 10, 64, 200, 0.01, None),   # C2 shape
    (340, [1024], 10, 32, 40, 1e-4, None),   # C4 shape
    (4, [8], 3, 12, 60, 0.1, None),          # C1 shape
    (13, [37], 41, 9, 30, 0.05, 5),          # ragged: I%4 != 0, C > 32, H % G != 0
    (6, [3], 2, 5, 17, 0.2, None),           # H < 8 warps, C == 2
    (784, [128], 10, 64, 1, 0.01, 16),       # a single step
])
@pytest.mark.parametrize("mode", ["cluster", "grid", "stream"])
def test_sgd_stream_fast_vs_oracle(lane, fast, monkeypatch, mode, F, H, C, n, steps, eta, ctas):
    # cluster: one thread-block cluster, DSMEM exchange; grid: all SMs, L2
    # exchange, W0 in shared memory; stream: grid with W0 streamed from HBM
    monkeypatch.setenv("LANE_B200_SGD_MODE", "cluster" if mode == "cluster" else "grid")
    if mode == "stream":
        monkeypatch.setenv("LANE_B200_SGD_STREAM", "1")
    if ctas:
        monkeypatch.setenv("LANE_B200_SGD_CLUSTER" if mode == "cluster" else "LANE_B200_SGD_CTAS",
                           str(min(ctas, 16)))
    X, T = po.synthetic_dataset(F, C, n, 9)
    order = np.random.default_rng(1).integers(0, n, steps).astype(np.uint32)
    net = lane.build_network(F, H, C, seed=42, device=fast)
    orc = po.OracleNet(F, H, C, seed=42)
    want_loss = orc.sgd_run(X, T, steps, eta, order=order)
    Xd, Td, Od = upload(fast, X), upload(fast, T), upload(fast, order, np.uint32)
    Ld = upload(fast, np.zeros(1, np.float64), np.float64)
    before = fast.kernel_launches
    net.sgd_stream(Xd, Td, n, steps, eta, order_dev=Od, loss_dev=Ld)
    fast.sync()
    if C <= 32:  # persistent plan: one kernel (+ G/DW materialisation)
        assert fast.kernel_launches - before <= 3
    loss = np.zeros(1, np.float64)
    fast.d2h(loss, Ld)
    assert abs(loss[0] - want_loss) <= 1e-4 * abs(want_loss)
    for l, layer in enumerate(net.layers):
        got, want = layer_arrays(layer), oracle_arrays(orc, l)
        for b in BUFS:
            rtol = 1e-5 if steps == 1 else 2e-4
            assert_close(got[b], want[b], rtol, f"layer {l} {b}")
    for p in (Xd, Td, Od, Ld):
        fast.free(p)


@pytest.mark.parametrize("F,H,C,n,steps,eta,D", [
    (784, [128], 10, 64, 200, 0.01, 3),     # C2 shape, partial last block
    (784, [128], 10, 64, 200, 0.01, 2),     # shortest lag
    (784, [128], 10, 64, 203, 0.01, 6),     # longest lag (window 95 rows)
    (340, [256], 10, 32, 70, 1e-3, 3),      # C4 H=256: 8 hidden units per chain lane
    (4, [8], 3, 12, 60, 0.1, 3),            # C1 shape: 2 producers, mostly idle lanes
    (20, [64], 16, 9, 45, 0.05, 3),         # 16 classes (the transpose-reduce limit)
    (33, [4], 7, 5, 33, 0.1, 3),            # one producer, I % 4 != 0
    (784, [128], 10, 64, 1, 0.01, 3),       # a single step
    (784, [128], 10, 64, 17, 0.01, 3),      # shorter than the window
    (340, [512], 10, 32, 60, 1e-3, 2),      # cluster chain: 4 chain CTAs x 128 units, DSMEM exchange
    (340, [1024], 10, 32, 60, 1e-3, 2),     # 8 chain CTAs, 2 column quads per producer
    (340, [2048], 10, 32, 45, 1e-3, 3),     # 16 chain CTAs (non-portable cluster), 4 quads per producer
    (340, [4096], 10, 32, 40, 1e-3, 2),     # 16 chain CTAs x 2 warps, W0 slices in producer smem
    (340, [4096], 10, 32, 50, 1e-3, 3),     # the same at the default lag of the 16-CTA chains
    (340, [8192], 10, 32, 40, 1e-3, 2),     # 16 chain CTAs x 4 warps, d0 straight to L2, 19 quads/producer
    (64, [384], 7, 16, 50, 0.02, 2),        # 4 chain CTAs x 96 units (partial slices)
    (784, [128], 10, 64, 150, 0.01, -2),    # two chain warps (2 units/lane) instead of one
    (100, [96], 10, 20, 90, 0.02, -3),      # two chain warps, H % 64 != 0
])
def test_sgd_window_fast_vs_oracle(lane, fast, monkeypatch, F, H, C, n, steps, eta, D):
    # delayed-base windowed kernel: chain CTA + W0 producer CTAs + banded Gram
    # (D < 0: lag |D| with the chain split over two warps)
    monkeypatch.setenv("LANE_B200_SGD_MODE", "window")
    monkeypatch.setenv("LANE_B200_SGD_WIN_D", str(abs(D)))
    if D < 0:
        monkeypatch.setenv("LANE_B200_SGD_WIN_NCW", "2")
    X, T = po.synthetic_dataset(F, C, n, 9)
    order = np.random.default_rng(2).integers(0, n, steps).astype(np.uint32)
    net = lane.build_network(F, H, C, seed=42, device=fast)
    orc = po.OracleNet(F, H, C, seed=42)
    want_loss = orc.sgd_run(X, T, steps, eta, order=order)
    Xd, Td, Od = upload(fast, X), upload(fast, T), upload(fast, order, np.uint32)
    Ld = upload(fast, np.zeros(1, np.float64), np.float64)
    Cd = upload(fast, np.zeros(1, np.uint64), np.uint64)
    before = fast.kernel_launches
    net.sgd_stream(Xd, Td, n, steps, eta, order_dev=Od, loss_dev=Ld, correct_dev=Cd)
    fast.sync()
    assert fast.kernel_launches - before == 4  # Gram pre-pass, window kernel, G/DW x2
    loss = np.zeros(1, np.float64)
    fast.d2h(loss, Ld)
    assert abs(loss[0] - want_loss) <= 1e-4 * abs(want_loss)
    for l, layer in enumerate(net.layers):
        got, want = layer_arrays(layer), oracle_arrays(orc, l)
        for b in BUFS:
            rtol = 1e-5 if steps == 1 else 2e-4
            assert_close(got[b], want[b], rtol, f"layer {l} {b}")
    for p in (Xd, Td, Od, Ld, Cd):
        fast.free(p)


def test_sgd_window_no_order_wraps_dataset(lane, fast, monkeypatch):
    # no order array: sample s is row s % n (stream longer than the dataset)
    monkeypatch.setenv("LANE_B200_SGD_MODE", "window")
    F, H, C, n, steps, eta = 50, [32], 10, 7, 40, 0.05
    X, T = po.synthetic_dataset(F, C, n, 9)
    net = lane.build_network(F, H, C, seed=42, device=fast)
    orc = po.OracleNet(F, H, C, seed=42)
    orc.sgd_run(X, T, steps, eta, order=(np.arange(steps) % n).astype(np.uint32))
    Xd, Td = upload(fast, X), upload(fast, T)
    net.sgd_stream(Xd, Td, n, steps, eta)
    fast.sync()
    for l, layer in enumerate(net.layers):
        got, want = layer_arrays(layer), oracle_arrays(orc, l)
        for b in BUFS:
            assert_close(got[b], want[b], 2e-4, f"layer {l} {b}")
    for p in (Xd, Td):
        fast.free(p)


# ----------------------------------------------------- train / evaluate -----

def iris():
    X, T = po.load_dataset(IRIS, 4, 3)
    return po.split(X, T, 0.9, 42)


def test_train_strict_iris_one_epoch_bitwise_vs_reference_golden(lane, strict):
    Xtr, Ttr, _, _ = iris()
    net = lane.build_network(4, [8], 3, seed=42, device=strict)
    st = lane.train(net, lane.DataSet(Xtr, Ttr),
                    lane.TrainerConfig(lane.LearningRate(0.1), 0.0, 1, 42))
    assert_bitwise([st[0].mean_loss, st[0].accuracy], GOLD["iris1_stats"], "epoch stats")
    assert net.hash() == int(GOLD["iris1_hash"][0])


def test_train_strict_xor_77_epochs(lane, strict):
    # proj/tests/test_training.cpp:204-221 regression oracle, bit-for-bit
    Xx = np.float32([[0, 0], [0, 1], [1, 0], [1, 1]])
    Tx = np.float32([[1, 0], [0, 1], [0, 1], [1, 0]])
    net = lane.build_network(2, [4], 2, seed=111, device=strict)
    st = lane.train(net, lane.DataSet(Xx, Tx), lane.TrainerConfig(lane.LearningRate(0.5), 0.05, 5000, 111))
    assert len(st) == 77
    assert_bitwise([s.mean_loss for s in st], GOLD["xor_curve"], "loss curve")
    assert lane.evaluate(net, lane.DataSet(Xx, Tx)).accuracy == 1.0


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_train_iris_acceptance_c5(lane, dev, mode):
    # proj/tests/acceptance.cpp:443-469: 135/15 split, hidden [8], acc >= 0.9
    dev.numerics = lane.NUMERICS_STRICT if mode == "strict" else lane.NUMERICS_FAST
    try:
        Xtr, Ttr, Xte, Tte = iris()
        net = lane.build_network(4, [8], 3, seed=42, device=dev)
        st = lane.train(net, lane.DataSet(Xtr, Ttr),
                        lane.TrainerConfig(lane.LearningRate(0.1), 0.05, 2000, 42))
        res = lane.evaluate(net, lane.DataSet(Xte, Tte))
        assert res.accuracy >= 0.9
        curve = np.array([s.mean_loss for s in st], np.float32)
        if mode == "strict":
            assert len(st) == int(GOLD["irisC5_epochs"][0])
            assert_bitwise(curve, GOLD["irisC5_curve"], "loss curve")
        else:
            ref = GOLD["irisC5_curve"]
            k = min(len(curve), len(ref))
            np.testing.assert_allclose(curve[:k], ref[:k], rtol=1e-4)
            assert abs(len(st) - len(ref)) <= 1
    finally:
        dev.numerics = lane.NUMERICS_FAST


def test_train_fast_c2_epoch_loss_curve(lane, fast):
    X, T = po.synthetic_dataset(784, 10, 2000, 9)
    net = lane.build_network(784, [128], 10, seed=42, device=fast)
    orc = po.OracleNet(784, [128], 10, seed=42)
    st = lane.train(net, lane.DataSet(X, T), lane.TrainerConfig(lane.LearningRate(0.01), 0.0, 2, 42))
    ref = orc.train(X, T, 0.01, max_epochs=2, seed=42)
    for g, r in zip(st, ref):
        assert abs(g.mean_loss - r[1]) <= 1e-4 * abs(r[1])
        assert abs(g.accuracy - r[2]) <= 2.0 / len(X)
    assert_close(net.hidden[0].weights, orc.get(0, po.W), 1e-4, "W0")


def test_train_rejects_empty_or_mismatched(lane, dev):
    net = lane.build_network(2, [4], 2, seed=3, device=dev)
    with pytest.raises(lane.TrainingError):
        lane.train(net, lane.DataSet(np.zeros((0, 2), np.float32), np.zeros((0, 2), np.float32)),
                   lane.TrainerConfig())
    with pytest.raises(lane.ShapeError):
        lane.train(net, lane.DataSet(np.zeros((4, 3), np.float32), np.eye(2, dtype=np.float32)[[0, 1, 0, 1]]),
                   lane.TrainerConfig())


def test_evaluate_ties_to_lowest_class(lane, dev):
    # proj/tests/test_training.cpp:282-300
    net = lane.FeedForwardNetwork(2, [], 3, device=dev)
    d = lane.DataSet(np.full((3, 2), 0.5, np.float32), np.eye(3, dtype=np.float32))
    np.testing.assert_allclose(lane.evaluate(net, d).accuracy, 1.0 / 3.0, rtol=1e-6)


# ---------------------------------------------------- mini-batch ext -------

def test_minibatch_b1_mu0_reduces_to_backward_plan(lane, fast):
    X, T = po.synthetic_dataset(24, 5, 3, 2)
    net = lane.build_network(24, [16, 12], 5, seed=9, device=fast, max_batch=4)
    orc = po.OracleNet(24, [16, 12], 5, seed=9)
    Xd, Td = upload(fast, X), upload(fast, T)
    for s in range(3):
        net.minibatch_step(Xd + s * 24 * 4, Td + s * 5 * 4, 1, 0.05, 0.0)
        orc.forward(X[s])
        orc.backward_plan_run(T[s], 0.05)
    for l, layer in enumerate(net.layers):
        assert_close(layer.weights, orc.get(l, po.W), 1e-5, f"W{l}")
        assert_close(layer.biases, orc.get(l, po.B), 1e-5, f"b{l}")
    fast.free(Xd)
    fast.free(Td)


@pytest.mark.parametrize("F,H,C,B,mu", [(64, [96, 80], 10, 32, 0.9), (130, [200], 7, 17, 0.0),
                                        (1024, [512, 512], 10, 64, 0.9)])
def test_minibatch_momentum_vs_oracle(lane, fast, F, H, C, B, mu):
    # 4 steps: eager (sizes the workspaces), graph capture, two graph replays
    X, T = po.synthetic_dataset(F, C, 4 * B, 4)
    net = lane.build_network(F, H, C, seed=1, device=fast, max_batch=B)
    orc = po.OracleNet(F, H, C, seed=1)
    Xd, Td = upload(fast, X), upload(fast, T)
    for s in range(4):
        net.minibatch_step(Xd + s * B * F * 4, Td + s * B * C * 4, B, 0.05, mu)
        orc.minibatch_step(X[s * B:(s + 1) * B], T[s * B:(s + 1) * B], 0.05, mu)
    for l, layer in enumerate(net.layers):
        assert_close(layer.gradients, orc.get(l, po.G), 1e-4, f"G{l}")
        assert_close(layer.delta_weights, orc.get(l, po.DW), 1e-4, f"DW{l}")
        assert_close(layer.weights, orc.get(l, po.W), 1e-5, f"W{l}")
    fast.free(Xd)
    fast.free(Td)


@pytest.mark.parametrize("shuffle,drop_last,n", [(False, True, 200), (True, True, 200), (True, False, 203)])
def test_train_minibatch_pipeline_matches_manual_steps(lane, fast, shuffle, drop_last, n):
    """The pipelined trainer (host gather -> pinned slot -> copy stream) runs
    exactly the steps a caller would run by hand on the same batches: bitwise
    identical weights, per-step losses equal to each step's own loss sum."""
    F, H, C, B, mu, eta, E = 40, [64, 48], 6, 16, 0.9, 0.05, 3
    X, T = po.synthetic_dataset(F, C, n, 5)
    a = lane.build_network(F, H, C, seed=3, device=fast, max_batch=B)
    b = lane.build_network(F, H, C, seed=3, device=fast, max_batch=B)
    means, steps = lane.train_minibatch(a, lane.DataSet(X, T), B, eta, mu, epochs=E, seed=42, shuffle=shuffle,
                                        drop_last=drop_last, step_losses=True)
    orders = po.shuffle_orders(n, E, 42) if shuffle else np.tile(np.arange(n, dtype=np.uint32), (E, 1))
    nb = n // B + (0 if drop_last or n % B == 0 else 1)
    assert steps.shape == (E, nb)
    ld = fast.alloc(8)
    Xd, Td = fast.alloc(B * F * 4), fast.alloc(B * C * 4)
    for e in range(E):
        for s in range(nb):
            idx = orders[e][s * B:(s + 1) * B]
            fast.h2d(Xd, np.ascontiguousarray(X[idx]))
            fast.h2d(Td, np.ascontiguousarray(T[idx]))
            fast.h2d(ld, np.zeros(1, np.float64))
            b.minibatch_step(Xd, Td, len(idx), eta, mu, ld)
            got = np.zeros(1, np.float64)
            fast.d2h(got, ld)
            np.testing.assert_allclose(steps[e, s], got[0] / len(idx), rtol=1e-5)
        np.testing.assert_allclose(means[e], steps[e] @ np.array(
            [min(B, n - s * B) for s in range(nb)], np.float64) / sum(min(B, n - s * B) for s in range(nb)),
            rtol=1e-5)
    for la, lb in zip(a.layers, b.layers):
        np.testing.assert_array_equal(la.weights, lb.weights)
        np.testing.assert_array_equal(la.delta_weights, lb.delta_weights)
    for p_ in (ld, Xd, Td):
        fast.free(p_)


def test_train_minibatch_from_loaded_dataset(lane, fast, tmp_path):
    """load_dataset (page-locked rows) -> split -> train_minibatch -> evaluate,
    the loss falling over the epochs (Iris, 4-16-3)."""
    import os
    iris = os.path.join(os.path.dirname(__file__), "golden", "iris_normalized.txt")
    tr, te = lane.split(lane.load_dataset(iris, 4, 3), 0.9, 42)
    net = lane.build_network(4, [16], 3, seed=42, device=fast, max_batch=16)
    means = lane.train_minibatch(net, tr, 16, 0.2, 0.9, epochs=60, seed=1)
    assert means[-1] < 0.5 * means[0]
    assert lane.evaluate(net, te).accuracy >= 0.8
    with pytest.raises(lane.ShapeError):
        lane.train_minibatch(net, tr, 17, 0.1)
    with pytest.raises(lane.TrainingError):
        lane.train_minibatch(net, lane.DataSet(tr.features[:8], tr.labels[:8]), 16, 0.1)


@pytest.mark.parametrize("F,H,C,want", [(784, [128], 10, "window"), (4, [8], 3, "window"),
                                        (340, [256], 10, "window"), (340, [1024], 10, "window"),
                                        (340, [2048], 10, "window"), (340, [1000], 10, "cluster"),
                                        (340, [4096], 10, "window"), (340, [8192], 10, "window"),
                                        (340, [16384], 10, "grid")])
def test_sgd_plan_selection(lane, fast, F, H, C, want):
    # the fused plan the headline shapes run (no silent fallback to layer kernels)
    net = lane.build_network(F, H, C, seed=42, device=fast)
    assert net.sgd_plan().split()[0] == want, net.sgd_plan()


@pytest.mark.parametrize("H,D", [(128, 2), (1024, 2), (2048, 3), (4096, 3), (8192, 2)])
def test_sgd_window_default_lag(lane, fast, monkeypatch, H, D):
    # the 16-CTA cluster chains take lag 3 where its rings fit (not at 8192)
    monkeypatch.delenv("LANE_B200_SGD_WIN_D", raising=False)
    net = lane.build_network(784 if H == 128 else 340, [H], 10, seed=42, device=fast)
    assert f" D={D} " in net.sgd_plan(), net.sgd_plan()


def test_sgd_window_long_stream_chunks(lane, fast, monkeypatch):
    # > 2^18 samples: the stream runs as several window launches (the banded
    # Gram scratch is per launch); state, loss and accuracy carry across
    monkeypatch.setenv("LANE_B200_SGD_MODE", "window")
    F, H, C, n, steps, eta = 4, [8], 3, 135, (1 << 18) + 1000, 0.01
    X, T = po.synthetic_dataset(F, C, n, 9)
    net = lane.build_network(F, H, C, seed=42, device=fast)
    orc = po.OracleNet(F, H, C, seed=42)
    order = np.random.default_rng(7).integers(0, n, steps).astype(np.uint32)
    want = orc.sgd_run(X, T, steps, eta, order=order)
    Xd, Td, Od = upload(fast, X), upload(fast, T), upload(fast, order, np.uint32)
    Ld = upload(fast, np.zeros(1, np.float64), np.float64)
    before = fast.kernel_launches
    net.sgd_stream(Xd, Td, n, steps, eta, order_dev=Od, loss_dev=Ld)
    fast.sync()
    assert fast.kernel_launches - before == 2 * 2 + 2  # 2 x (Gram + window) + G/DW x2
    loss = np.zeros(1, np.float64)
    fast.d2h(loss, Ld)
    assert abs(loss[0] - want) <= 1e-4 * abs(want)
    # 262k chaotic SGD steps: the weights agree loosely, the loss tightly
    for l, layer in enumerate(net.layers):
        assert_close(layer.weights, orc.get(l, po.W), 2e-3, f"W{l}")
    for p in (Xd, Td, Od, Ld):
        fast.free(p)


# ------------------------------------------- finite-difference gradients ---

def _ce_loss64(Ws, bs, X, T):
    """Mean cross entropy in float64 (proj/tests/acceptance.cpp:62-98, ce_loss_double)."""
    a = np.asarray(X, np.float64)
    for W, b in zip(Ws[:-1], bs[:-1]):
        a = np.tanh(a @ W + b)
    z = a @ Ws[-1] + bs[-1]
    z = z - z.max(axis=-1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=-1, keepdims=True))
    return float(-(np.asarray(T, np.float64) * logp).sum(axis=-1).mean())


def _fd_check(Ws, bs, X, T, l, G, gb):
    """acceptance.cpp:100-140: central differences, h = 1e-3 max(1, |w|), rel 1e-3."""
    worst = 0.0
    for P, A in ((Ws[l], G), (bs[l], gb)):
        for idx in np.ndindex(P.shape):
            saved = P[idx]
            h = 1e-3 * max(1.0, abs(saved))
            P[idx] = saved + h
            up = _ce_loss64(Ws, bs, X, T)
            P[idx] = saved - h
            dn = _ce_loss64(Ws, bs, X, T)
            P[idx] = saved
            fd = (up - dn) / (2 * h)
            rel = abs(A[idx] - fd) / max(1.0, abs(A[idx]), abs(fd))
            worst = max(worst, rel)
    assert worst <= 1e-3, worst
    return worst


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_layer_gradients_vs_finite_differences(lane, dev, mode):
    """The reference's gradient-correctness criterion (acceptance.cpp:142-162)
    on the GPU layer API: 20 networks up to 8-8-4, every weight and bias of
    both layers, analytic G / delta against float64 central differences."""
    dev.numerics = lane.NUMERICS_STRICT if mode == "strict" else lane.NUMERICS_FAST
    try:
        rs = np.random.default_rng(4242)
        for trial in range(20):
            F, H, C_ = 1 + int(rs.integers(8)), 1 + int(rs.integers(8)), 2 + int(rs.integers(3))
            net = lane.build_network(F, [H], C_, seed=int(rs.integers(1 << 30)), device=dev)
            x = rs.uniform(-1, 1, F).astype(np.float32)
            t = np.eye(C_, dtype=np.float32)[int(rs.integers(C_))]
            net.forward(x)
            net.output.backward(t, 0.01)
            net.hidden[0].backward(eta=0.01)
            Ws = [net.hidden[0].weights.astype(np.float64), net.output.weights.astype(np.float64)]
            bs = [net.hidden[0].biases.astype(np.float64), net.output.biases.astype(np.float64)]
            for l, layer in enumerate([net.hidden[0], net.output]):
                _fd_check(Ws, bs, x[None], t[None], l, layer.gradients.astype(np.float64),
                          layer.deltas.astype(np.float64))
    finally:
        dev.numerics = lane.NUMERICS_FAST


def test_minibatch_gradients_vs_finite_differences(lane, fast):
    """Mini-batch extension ("FD of the mean loss"): the mean
    gradient the step applies, read back as G / BIAS_GRAD, against float64
    central differences of the batch-mean cross entropy at the pre-update
    weights."""
    F, H, C_, B = 6, [7, 5], 3, 9
    X, T = po.synthetic_dataset(F, C_, B, 3)
    net = lane.build_network(F, H, C_, seed=11, device=fast, max_batch=B)
    Ws = [L.weights.astype(np.float64) for L in net.layers]
    bs = [L.biases.astype(np.float64) for L in net.layers]
    Xd, Td = upload(fast, X), upload(fast, T)
    net.minibatch_step(Xd, Td, B, 0.05, 0.0)
    for l, L in enumerate(net.layers):
        G = L.gradients.astype(np.float64)
        gb = L.read(lane.BIAS_GRAD).astype(np.float64)
        _fd_check(Ws, bs, X, T, l, G, gb)
    fast.free(Xd)
    fast.free(Td)


@pytest.mark.parametrize("F,H,C,n", [(784, [128], 10, 3000), (64, [96, 80], 7, 500), (130, [33], 3, 257)])
def test_evaluate_batched_fast_vs_oracle(lane, fast, F, H, C, n):
    """FAST evaluate runs the forward of whole row chunks as GEMMs; mean loss
    and accuracy against the oracle's per-sample evaluate (network.cpp:184-204)
    after a short training run moved the weights off their init."""
    X, T = po.synthetic_dataset(F, C, n, 21)
    net = lane.build_network(F, H, C, seed=5, device=fast)
    orc = po.OracleNet(F, H, C, seed=5)
    lane.train(net, lane.DataSet(X, T), lane.TrainerConfig(lane.LearningRate(0.01), 0.0, 1, 3))
    for l, layer in enumerate(net.layers):  # same weights on both sides
        orc.set(l, po.W, layer.weights)
        orc.set(l, po.B, layer.biases)
    got = lane.evaluate(net, lane.DataSet(X, T))
    loss, acc = orc.evaluate(X, T)
    assert abs(got.mean_loss - loss) <= 1e-5 * abs(loss) + 1e-7
    assert abs(got.accuracy - acc) <= 2.0 / n


def test_nccl_communicator_single_rank(lane):
    """The data-parallel plumbing on the one GPU available: an NCCL
    communicator of one rank (id created in the library), mini-batch steps
    through it, and results bitwise equal to a context without one."""
    from paper_2001_04206_b200 import parallel
    F, H, C_, B = 48, [64], 5, 32
    X, T = po.synthetic_dataset(F, C_, 2 * B, 6)
    out = []
    for use_comm in (False, True):
        d = lane.Device(0)
        if use_comm:
            parallel.init_comm(d, 0, 1)
            assert d.world == 1
        net = lane.build_network(F, H, C_, seed=8, device=d, max_batch=B)
        Xd, Td = upload(d, X), upload(d, T)
        for s in range(2):
            net.minibatch_step(Xd + s * B * F * 4, Td + s * B * C_ * 4, B, 0.05, 0.9)
        net.allreduce_grads()  # a no-op sum over one rank
        out.append([layer.weights.copy() for layer in net.layers])
        if use_comm:
            d.comm_destroy()
        d.free(Xd)
        d.free(Td)
        net.close()
        d.close()
    for a, b in zip(*out):
        np.testing.assert_array_equal(a, b)


def test_nccl_bucketed_allreduce_path_single_rank():
    """The data-parallel step's per-layer allreduces on a communication stream
    (overlapping the remaining wgrads, captured in the step graph), forced on
    a one-rank communicator: weights bitwise equal to the plain step."""
    import subprocess
    import sys
    code = r'''
import numpy as np
from oracle import pyoracle as po
from paper_2001_04206_b200 import lane, parallel
F, H, C, B = 40, [64, 48], 6, 32
X, T = po.synthetic_dataset(F, C, 4 * B, 7)
out = []
for use_comm in (False, True):
    d = lane.Device(0)
    if use_comm:
        parallel.init_comm(d, 0, 1)
    net = lane.build_network(F, H, C, seed=9, device=d, max_batch=B)
    xd, td = d.alloc(X.nbytes), d.alloc(T.nbytes)
    d.h2d(xd, X)
    d.h2d(td, T)
    for s in range(4):  # eager, capture, two graph replays
        net.minibatch_step(xd + s * B * F * 4, td + s * B * C * 4, B, 0.05, 0.9)
    d.sync()
    out.append([L.weights.copy() for L in net.layers] + [L.biases.copy() for L in net.layers])
for a, b in zip(*out):
    assert np.array_equal(a, b)
print("BUCKETS OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LANE_B200_MB_BUCKETS="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "BUCKETS OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def _random_window_shapes(count=10, seed=20261017):
    rs = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        F = int(rs.integers(3, 900))
        H = int(rs.choice([4, 8, 12, 16, 32, 60, 96, 124, 128]))
        C_ = int(rs.integers(2, 17))
        n = int(rs.integers(5, 90))
        steps = int(rs.integers(1, 260))
        out.append((F, H, C_, n, steps))
    return out


@pytest.mark.parametrize("F,H,C,n,steps", _random_window_shapes())
def test_sgd_stream_random_shapes_vs_oracle(lane, fast, F, H, C, n, steps):
    """Seeded random shapes through the default fused plan (the window kernel
    for H <= 128): odd feature widths, 2..16 classes, streams shorter and
    longer than the dataset, against the oracle's per-sample SGD."""
    X, T = po.synthetic_dataset(F, C, n, 13)
    eta = 0.01 if F > 100 else 0.05
    net = lane.build_network(F, [H], C, seed=7, device=fast)
    orc = po.OracleNet(F, [H], C, seed=7)
    want_loss = orc.sgd_run(X, T, steps, eta)
    Xd, Td = upload(fast, X), upload(fast, T)
    Ld = upload(fast, np.zeros(1, np.float64), np.float64)
    net.sgd_stream(Xd, Td, n, steps, eta, loss_dev=Ld)
    fast.sync()
    loss = np.zeros(1, np.float64)
    fast.d2h(loss, Ld)
    assert abs(loss[0] - want_loss) <= 1e-4 * abs(want_loss) + 1e-6
    for l, layer in enumerate(net.layers):
        assert_close(layer.weights, orc.get(l, po.W), 2e-4, f"W{l}")
        assert_close(layer.biases, orc.get(l, po.B), 2e-4, f"b{l}")
    fast.free(Xd)
    fast.free(Td)
    fast.free(Ld)


def _random_wide_shapes(count=8, seed=777):
    rs = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        F = int(rs.integers(8, 400))
        H = int(rs.choice([200, 256, 384, 512, 1000, 1024, 2048, 3000, 4096, 8192, 12288]))
        C_ = int(rs.integers(2, 11))
        n = int(rs.integers(5, 40))
        steps = int(rs.integers(20, 120))
        out.append((F, H, C_, n, steps))
    return out


@pytest.mark.parametrize("F,H,C,n,steps", _random_wide_shapes())
def test_sgd_stream_random_wide_shapes_vs_oracle(lane, fast, F, H, C, n, steps):
    """Seeded random wide layers through whichever fused plan the library picks
    (cluster-split window chains, the single-cluster kernel, the grid kernel)."""
    X, T = po.synthetic_dataset(F, C, n, 17)
    eta = 1e-3
    net = lane.build_network(F, [H], C, seed=3, device=fast)
    assert net.sgd_plan().split()[0] in ("window", "cluster", "grid"), net.sgd_plan()
    orc = po.OracleNet(F, [H], C, seed=3)
    want_loss = orc.sgd_run(X, T, steps, eta)
    Xd, Td = upload(fast, X), upload(fast, T)
    Ld = upload(fast, np.zeros(1, np.float64), np.float64)
    net.sgd_stream(Xd, Td, n, steps, eta, loss_dev=Ld)
    fast.sync()
    loss = np.zeros(1, np.float64)
    fast.d2h(loss, Ld)
    assert abs(loss[0] - want_loss) <= 1e-4 * abs(want_loss) + 1e-6
    for l, layer in enumerate(net.layers):
        assert_close(layer.weights, orc.get(l, po.W), 2e-4, f"W{l}")
        assert_close(layer.biases, orc.get(l, po.B), 2e-4, f"b{l}")
    fast.free(Xd)
    fast.free(Td)
    fast.free(Ld)


def _random_minibatch_shapes(count=10, seed=4096):
    rs = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        F = int(rs.choice([7, 33, 64, 130, 256, 515, 1024]))
        H = [int(rs.choice([5, 64, 96, 129, 256, 384, 640])) for _ in range(int(rs.integers(1, 3)))]
        C_ = int(rs.integers(2, 17))
        B = int(rs.choice([1, 3, 16, 64, 100, 256]))
        mu = float(rs.choice([0.0, 0.9]))
        out.append((F, H, C_, B, mu))
    return out


@pytest.mark.parametrize("F,H,C,B,mu", _random_minibatch_shapes())
def test_minibatch_random_shapes_vs_oracle(lane, fast, F, H, C, B, mu):
    """Seeded random widths and batches through the mini-batch step (tensor-core
    GEMMs where eligible, SIMT/skinny kernels elsewhere), three steps against
    the oracle's mini-batch restatement."""
    X, T = po.synthetic_dataset(F, C, 3 * B, 23)
    net = lane.build_network(F, H, C, seed=4, device=fast, max_batch=B)
    orc = po.OracleNet(F, H, C, seed=4)
    Xd, Td = upload(fast, X), upload(fast, T)
    for s in range(3):
        net.minibatch_step(Xd + s * B * F * 4, Td + s * B * C * 4, B, 0.03, mu)
        orc.minibatch_step(X[s * B:(s + 1) * B], T[s * B:(s + 1) * B], 0.03, mu)
    for l, layer in enumerate(net.layers):
        assert_close(layer.weights, orc.get(l, po.W), 1e-5, f"W{l}")
        assert_close(layer.biases, orc.get(l, po.B), 1e-5, f"b{l}")
        assert_close(layer.gradients, orc.get(l, po.G), 2e-4, f"G{l}")
    fast.free(Xd)
    fast.free(Td)


@pytest.mark.parametrize("F,H,C", [(4, [8], 3), (2, [4], 2), (32, [32], 16), (17, [13], 5)])
def test_sgd_tiny_stream_bitwise_vs_oracle(lane, strict, F, H, C):
    """STRICT: the one-warp tiny-net kernel computes in the reference's
    order, so a 200-sample stream (with an order permutation) equals the
    oracle's per-sample BackwardPlan::run bit for bit -- every LayerState
    buffer and the loss sum."""
    X, T = po.synthetic_dataset(F, C, 50, 5)
    net = lane.build_network(F, H, C, seed=3, device=strict)
    assert net.sgd_plan().split()[0] == "tiny"
    orc = po.OracleNet(F, H, C, seed=3)
    rs = np.random.default_rng(F * 100 + H[0])
    order = rs.integers(0, 50, 200).astype(np.uint32)
    dev = strict
    xd, td, od, ld = dev.alloc(X.nbytes), dev.alloc(T.nbytes), dev.alloc(order.nbytes), dev.alloc(16)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    dev.h2d(od, order)
    dev.h2d(ld, np.zeros(2, np.float64))
    net.sgd_stream(xd, td, 50, 200, 0.05, order_dev=od, loss_dev=ld, correct_dev=ld + 8)
    dev.sync()
    want = orc.sgd_run(X, T, 200, 0.05, order)  # loss sum in sample order, double
    st = np.zeros(2, np.float64)
    dev.d2h(st, ld)
    assert st[0] == want, (st[0], want)
    assert net.hash() == orc.hash(), "tiny stream not bit-identical to the reference order"
    for li, layer in enumerate(net.layers):
        for buf in BUFS:
            assert_bitwise(getattr(layer, buf), orc.get(li, BUFS.index(buf)), f"layer {li} {buf}")
    for p_ in (xd, td, od, ld):
        dev.free(p_)



@pytest.mark.parametrize("F,H,C,want", [(4, [8], 3, "tiny"), (2, [4], 2, "tiny"), (32, [32], 16, "tiny"),
                                        (33, [32], 16, "layer"), (784, [128], 10, "layer")])
def test_sgd_plan_selection_strict(lane, strict, F, H, C, want):
    # STRICT: tiny nets run the one-warp reference-order kernel, the rest the layer path
    net = lane.build_network(F, H, C, seed=42, device=strict)
    assert net.sgd_plan().split()[0] == want, net.sgd_plan()
