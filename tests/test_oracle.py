"""Pin the C restatement (oracle/lane_oracle.c) before trusting it as the checker.

1. Against tests/golden/golden.npz -- produced by the unmodified reference
   library (tests/golden/make_golden.py) -- bit-for-bit.  Runs everywhere.
2. Against the reference's own test KATs (values cited from proj/tests).
3. Live against oracle/_ref/liblane_ref.so on fresh random cases, when the
   reference was built here (skipped on the GPU box, where it may be absent).
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
IRIS = os.path.join(os.path.dirname(__file__), "golden", "iris_normalized.txt")
needs_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(a, b):
    np.testing.assert_array_equal(bits(a), bits(b))


# ------------------------------------------------------------------ rng ---

def test_splitmix_seed42_kat():
    # proj/tests/test_tensor.cpp:115-125
    x, _ = po.synthetic_dataset(4, 2, 1, 42)
    assert x[0].tolist() == [float.fromhex("0x1.7bae64p-1"), float.fromhex("0x1.477f18p-3"),
                             float.fromhex("0x1.1d499cp-2"), float.fromhex("0x1.607384p-2")]
    assert_bitwise(x[0], GOLD["rng_fill_42_unit"])


@pytest.mark.parametrize("seed", [42, 7, 0, 2026])
def test_rng_streams_match_golden(seed):
    import ctypes as C
    L = po.oracle_lib()
    st = (C.c_uint64 * 2)()
    L.lo_rng_init(C.cast(st, C.c_void_p), seed)
    got = np.array([L.lo_rng_next_u64(C.cast(st, C.c_void_p)) for _ in range(16)], np.uint64)
    np.testing.assert_array_equal(got, GOLD[f"rng_u64_{seed}"])
    L.lo_rng_init(C.cast(st, C.c_void_p), seed)
    v = np.zeros(16, np.float32)
    L.lo_random_fill(v, 16, C.cast(st, C.c_void_p), -0.5, 0.5)
    assert_bitwise(v, GOLD[f"rng_fill_{seed}"])


# --------------------------------------------------------- layer KATs ---

def test_softmax_backward_hand_kat():
    # proj/tests/test_layers.cpp:125-142
    r = po.oracle_layer_backward("softmax", [0.7, 0.3], [2.0], 0.1, target=[1.0, 0.0])
    np.testing.assert_allclose(r["deltas"], [-0.3, 0.3], rtol=1e-6)
    np.testing.assert_allclose(r["gradients"][0], [-0.6, 0.6], rtol=1e-6)
    np.testing.assert_allclose(r["delta_weights"][0], [0.06, -0.06], rtol=1e-6)
    np.testing.assert_allclose(r["delta_biases"], [0.03, -0.03], rtol=1e-6)


def test_softmax_backward_zero_signal():
    # proj/tests/test_layers.cpp:144-161
    r = po.oracle_layer_backward("softmax", [0, 1, 0], [0.4, -0.2], 0.5, target=[0, 1, 0])
    for v in r.values():
        assert not np.any(v)


def test_fc_backward_hand_kat():
    # proj/tests/test_layers.cpp:209-222: (1 - 0.25) * 0.2 * 3.0 = 0.45
    r = po.oracle_layer_backward("fc", [0.5], [1.0], 0.1, next_W=[[3.0]], next_d=[0.2])
    np.testing.assert_allclose(r["deltas"], [0.45], rtol=1e-6)


def test_fc_backward_zero_next_deltas():
    # proj/tests/test_layers.cpp:224-238
    r = po.oracle_layer_backward("fc", [0.3, -0.2, 0.9], [0.5, -0.5], 0.1,
                                 next_W=np.ones((3, 2)), next_d=[0.0, 0.0])
    assert not np.any(r["deltas"]) and not np.any(r["gradients"])


def test_apply_updates_kat():
    # proj/tests/test_layers.cpp:240-258 (through a 1-1-2 network's hidden layer)
    net = po.OracleNet(1, [1], 2)
    net.set(0, po.W, [1.0])
    net.set(0, po.DW, [-0.06])
    net.set(0, po.DELTA_BIASES, [0.5])
    import ctypes as C
    lay = C.byref(net._p.contents.layers[0])
    po.oracle_lib().lo_apply_updates(lay)
    assert net.get(0, po.W)[0] == np.float32(0.94)
    assert net.get(0, po.B)[0] == np.float32(0.5)
    po.oracle_lib().lo_apply_updates(lay)  # additive
    np.testing.assert_allclose(net.get(0, po.W)[0], 0.88, rtol=1e-6)


def test_cross_entropy_kats():
    # proj/tests/test_training.cpp:89-101
    ce = lambda p, t: po.oracle_lib().lo_cross_entropy(np.float32(p), np.float32(t), len(p))
    assert ce([0, 1, 0], [0, 1, 0]) <= 1e-9
    np.testing.assert_allclose(ce([1 / 3] * 3, [1, 0, 0]), np.log(3.0), rtol=1e-6)
    np.testing.assert_allclose(ce([0, 1], [1, 0]), 27.631, rtol=1e-3)


# ------------------------------------------------- restatement == golden ---

@pytest.mark.parametrize("c", range(24))
def test_softmax_backward_matches_reference_golden(c):
    I, O = GOLD[f"smb{c}_shape"]
    v = GOLD[f"smb{c}_in"]
    r = po.oracle_layer_backward("softmax", v[:O], v[O:O + I], 0.05, target=v[O + I:])
    for k in ("deltas", "gradients", "delta_weights", "delta_biases"):
        assert_bitwise(r[k], GOLD[f"smb{c}_{k}"])


@pytest.mark.parametrize("c", range(24))
def test_fc_backward_matches_reference_golden(c):
    I, O, N = GOLD[f"fcb{c}_shape"]
    v = GOLD[f"fcb{c}_in"]
    r = po.oracle_layer_backward("fc", v[:O], v[O:O + I], 0.05,
                                 next_W=v[O + I:O + I + O * N].reshape(O, N),
                                 next_d=v[O + I + O * N:])
    for k in ("deltas", "gradients", "delta_weights", "delta_biases"):
        assert_bitwise(r[k], GOLD[f"fcb{c}_{k}"])


@pytest.mark.parametrize("c", range(16))
def test_layer_forward_matches_reference_golden(c):
    kind = "softmax" if c % 2 else "fc"
    z, a = po.oracle_layer_forward(kind, GOLD[f"fwd{c}_W"], GOLD[f"fwd{c}_b"], GOLD[f"fwd{c}_x"])
    assert_bitwise(z, GOLD[f"fwd{c}_z"])
    assert_bitwise(a, GOLD[f"fwd{c}_a"])


@pytest.mark.parametrize("name,F,H,C,eta,steps", [
    ("c1", 4, [8], 3, 0.01, 4), ("c2", 784, [128], 10, 0.01, 3),
    ("c4", 340, [256], 10, 1e-4, 2), ("deep", 16, [12, 9], 5, 0.05, 4)])
def test_network_steps_match_reference_golden(name, F, H, C, eta, steps):
    X, T = po.synthetic_dataset(F, C, 8, 9)
    net = po.OracleNet(F, H, C, seed=42)
    assert net.hash() == int(GOLD[f"{name}_hash0"][0])
    for s in range(steps):
        assert_bitwise(net.forward(X[s]), GOLD[f"{name}_probs"][s])
        net.backward_plan_run(T[s], eta)
        assert net.hash() == int(GOLD[f"{name}_hashes"][s]), f"step {s}"
        d = np.concatenate([net.get(l, po.DELTAS) for l in range(len(H) + 1)])
        assert_bitwise(d, GOLD[f"{name}_deltas"][s])


def iris_split():
    X, T = po.load_dataset(IRIS, 4, 3)
    assert X.shape == (150, 4)
    return po.split(X, T, 0.9, 42)


def test_iris_one_epoch_matches_reference_golden():
    Xtr, Ttr, _, _ = iris_split()
    assert len(Xtr) == 135
    net = po.OracleNet(4, [8], 3, seed=42)
    st = net.train(Xtr, Ttr, 0.1, max_epochs=1, seed=42)
    assert_bitwise(np.array(st[0][1:], np.float32), GOLD["iris1_stats"])
    assert net.hash() == int(GOLD["iris1_hash"][0])
    assert_bitwise(net.get(0, po.W), GOLD["iris1_W0"])


def test_iris_acceptance_c5_matches_reference_golden():
    # proj/tests/acceptance.cpp:443-469
    Xtr, Ttr, Xte, Tte = iris_split()
    net = po.OracleNet(4, [8], 3, seed=42)
    st = net.train(Xtr, Ttr, 0.1, max_epochs=2000, max_error=0.05, seed=42)
    assert len(st) == int(GOLD["irisC5_epochs"][0])
    assert_bitwise(np.array([s[1] for s in st], np.float32), GOLD["irisC5_curve"])
    acc = net.evaluate(Xte, Tte)[1]
    assert acc >= 0.9 and acc == GOLD["irisC5_test"][1]


def test_xor_regression_oracle_77_epochs():
    # proj/tests/test_training.cpp:204-221 ("recorded 77")
    Xx = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.float32)
    Tx = np.array([[1, 0], [0, 1], [0, 1], [1, 0]], np.float32)
    net = po.OracleNet(2, [4], 2, seed=111)
    st = net.train(Xx, Tx, 0.5, max_epochs=5000, max_error=0.05, seed=111)
    assert len(st) == 77 == int(GOLD["xor_epochs"][0])
    assert_bitwise(np.array([s[1] for s in st], np.float32), GOLD["xor_curve"])
    assert net.evaluate(Xx, Tx)[1] == 1.0


def test_minibatch_extension_reduces_to_reference_step():
    # B=1, mu=0 is bit-identical to BackwardPlan::run
    X, T = po.synthetic_dataset(20, 4, 3, 5)
    a = po.OracleNet(20, [16, 8], 4, seed=3)
    b = a.clone()
    for s in range(3):
        a.forward(X[s])
        a.backward_plan_run(T[s], 0.05)
        b.minibatch_step(X[s:s + 1], T[s:s + 1], 0.05, 0.0)
        assert a.hash() == b.hash()


# ------------------------------------------------ live vs the reference ---

@needs_ref
def test_live_random_networks_match_reference():
    rs = np.random.default_rng(7)
    for trial in range(12):
        F = int(rs.integers(1, 40))
        H = [int(rs.integers(1, 40)) for _ in range(int(rs.integers(0, 3)))]
        C = int(rs.integers(2, 8))
        seed = int(rs.integers(0, 2**63))
        ref, orc = po.RefNet(F, H, C, seed), po.OracleNet(F, H, C, seed)
        X, T = po.synthetic_dataset(F, C, 5, seed ^ 1)
        for s in range(5):
            assert_bitwise(ref.forward(X[s]), orc.forward(X[s]))
            ref.backward_plan_run(T[s], 0.03)
            orc.backward_plan_run(T[s], 0.03)
            for l in range(len(H) + 1):
                for buf in range(9):
                    assert_bitwise(ref.get(l, buf), orc.get(l, buf))


@needs_ref
def test_live_train_matches_reference_serial_and_parallel():
    X, T = po.synthetic_dataset(12, 3, 40, 11)
    for parallel in (False, True):
        ref, orc = po.RefNet(12, [20], 3, 5), po.OracleNet(12, [20], 3, 5)
        a = ref.train(X, T, 0.05, max_epochs=3, seed=9, parallel=parallel, workers=4)
        b = orc.train(X, T, 0.05, max_epochs=3, seed=9)
        assert a == [(e, float(np.float32(l)), float(np.float32(c))) for e, l, c in b]
        assert ref.hash() == orc.hash()


@needs_ref
def test_live_dataset_helpers_match_reference():
    X, T = po.load_dataset(IRIS, 4, 3)
    Xr = np.zeros((150, 4), np.float32)
    Tr = np.zeros((150, 3), np.float32)
    assert po.ref_lib().lr_load_dataset(IRIS.encode(), 4, 3, Xr.reshape(-1), Tr.reshape(-1),
                                       150) == 150
    assert_bitwise(X, Xr)
    Xo = np.zeros_like(Xr)
    To = np.zeros_like(Tr)
    ntr = po.ref_lib().lr_split(Xr.reshape(-1), Tr.reshape(-1), 150, 4, 3, 0.9, 42,
                                Xo.reshape(-1), To.reshape(-1))
    Xtr, Ttr, Xte, Tte = po.split(X, T, 0.9, 42)
    assert ntr == 135
    assert_bitwise(np.concatenate([Xtr, Xte]), Xo)
