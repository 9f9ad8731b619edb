"""ctypes front-end for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  It wraps

* ``oracle/build/liblane_oracle.so`` -- the plain-C restatement
  (``oracle/lane_oracle.c``), always available (built with gcc on demand);
* ``oracle/_ref/liblane_ref.so`` -- the unmodified reference library compiled
  from ``/root/reference/proj/src`` (``oracle/Makefile``); present wherever
  ``__graft_entry__.build()`` ran in the container that has the reference.

Buffer ids match ``include/lane_b200.h``: 0 W, 1 G, 2 DW, 3 b, 4 inputs,
5 netin, 6 outputs, 7 deltas, 8 delta_biases.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liblane_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblane_ref.so")

W, G, DW, B, INPUTS, NETIN, OUTPUTS, DELTAS, DELTA_BIASES = range(9)

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_szp = C.POINTER(C.c_size_t)


def build() -> None:
    """Compile the restatement (and the reference, where its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Layer(C.Structure):
    _fields_ = [("in_", C.c_size_t), ("out", C.c_size_t)] + [
        (n, C.POINTER(C.c_float)) for n in ("W", "G", "DW", "b", "x", "z", "a", "d", "db")
    ]


class _Net(C.Structure):
    _fields_ = [("input_width", C.c_size_t), ("n_hidden", C.c_size_t),
                ("layers", C.POINTER(_Layer))]


class _Stats(C.Structure):
    _fields_ = [("epoch", C.c_size_t), ("mean_loss", C.c_float), ("accuracy", C.c_float)]


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.lo_net_new.restype = C.POINTER(_Net)
        L.lo_net_new.argtypes = [C.c_size_t, _szp, C.c_size_t, C.c_size_t, C.c_uint64]
        L.lo_net_clone.restype = C.POINTER(_Net)
        L.lo_net_clone.argtypes = [C.POINTER(_Net)]
        L.lo_net_delete.argtypes = [C.POINTER(_Net)]
        L.lo_net_buf.restype = C.POINTER(C.c_float)
        L.lo_net_buf.argtypes = [C.POINTER(_Net), C.c_size_t, C.c_int, _szp]
        L.lo_net_forward.restype = C.POINTER(C.c_float)
        L.lo_net_forward.argtypes = [C.POINTER(_Net), _f32p]
        L.lo_backward_plan_run.argtypes = [C.POINTER(_Net), _f32p, C.c_float]
        L.lo_backward_no_update.argtypes = [C.POINTER(_Net), _f32p, C.c_float]
        L.lo_train.restype = C.c_size_t
        L.lo_train.argtypes = [C.POINTER(_Net), _f32p, _f32p, C.c_size_t, C.c_float, C.c_float,
                               C.c_size_t, C.c_uint64, C.POINTER(_Stats)]
        L.lo_evaluate.restype = _Stats
        L.lo_evaluate.argtypes = [C.POINTER(_Net), _f32p, _f32p, C.c_size_t]
        L.lo_sgd_run.restype = C.c_double
        L.lo_sgd_run.argtypes = [C.POINTER(_Net), _f32p, _f32p, C.c_size_t, C.c_void_p,
                                 C.c_size_t, C.c_float]
        L.lo_minibatch_step.restype = C.c_double
        L.lo_minibatch_step.argtypes = [C.POINTER(_Net), _f32p, _f32p, C.c_size_t, C.c_float,
                                        C.c_float]
        L.lo_net_hash.restype = C.c_uint64
        L.lo_net_hash.argtypes = [C.POINTER(_Net)]
        L.lo_cross_entropy.restype = C.c_float
        L.lo_cross_entropy.argtypes = [_f32p, _f32p, C.c_size_t]
        L.lo_synthetic_dataset.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, _f32p,
                                           _f32p]
        L.lo_load_dataset.restype = C.c_long
        L.lo_load_dataset.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, _f32p, _f32p,
                                      C.c_size_t]
        L.lo_split_order.restype = C.c_size_t
        L.lo_split_order.argtypes = [C.c_size_t, C.c_double, C.c_uint64, _u32p]
        L.lo_layer_new.restype = C.POINTER(_Layer)
        L.lo_layer_new.argtypes = [C.c_size_t, C.c_size_t]
        L.lo_layer_delete.argtypes = [C.POINTER(_Layer)]
        for fn in ("lo_fc_forward", "lo_softmax_forward"):
            getattr(L, fn).argtypes = [C.POINTER(_Layer), _f32p]
        L.lo_softmax_backward.argtypes = [C.POINTER(_Layer), _f32p, C.c_float]
        L.lo_fc_backward.argtypes = [C.POINTER(_Layer), _f32p, C.c_size_t, _f32p, C.c_float]
        L.lo_apply_updates.argtypes = [C.POINTER(_Layer)]
        L.lo_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        L.lo_random_fill.argtypes = [_f32p, C.c_size_t, C.c_void_p, C.c_float, C.c_float]
        L.lo_rng_next_u64.restype = C.c_uint64
        L.lo_rng_next_u64.argtypes = [C.c_void_p]
        L.lo_rng_below.restype = C.c_size_t
        L.lo_rng_below.argtypes = [C.c_void_p, C.c_size_t]
        L.lo_enlarge.argtypes = [_f32p, _f32p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.c_float, C.c_void_p, _f32p, _f32p]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; run make -C oracle)")
        L = C.CDLL(REF_SO)
        L.lr_last_error.restype = C.c_char_p
        L.lr_net_create.restype = C.c_void_p
        L.lr_net_create.argtypes = [C.c_size_t, _szp, C.c_size_t, C.c_size_t, C.c_uint64]
        L.lr_net_destroy.argtypes = [C.c_void_p]
        L.lr_net_rw.restype = C.c_long
        L.lr_net_rw.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_int]
        L.lr_net_forward.argtypes = [C.c_void_p, _f32p, _f32p]
        L.lr_backward_plan_run.argtypes = [C.c_void_p, _f32p, C.c_float, C.c_int, C.c_uint,
                                           C.c_void_p]
        L.lr_softmax_backward.argtypes = [C.c_size_t, C.c_size_t, _f32p, _f32p, _f32p, C.c_size_t,
                                          C.c_float, _f32p, _f32p, _f32p, _f32p]
        L.lr_fc_backward.argtypes = [C.c_size_t, C.c_size_t, _f32p, _f32p, C.c_size_t, C.c_size_t,
                                     _f32p, _f32p, C.c_size_t, C.c_float, _f32p, _f32p, _f32p,
                                     _f32p]
        L.lr_layer_forward.argtypes = [C.c_int, C.c_size_t, C.c_size_t, _f32p, _f32p, _f32p,
                                       _f32p, _f32p]
        L.lr_train.argtypes = [C.c_void_p, _f32p, _f32p, C.c_size_t, C.c_float, C.c_float,
                               C.c_size_t, C.c_uint64, C.c_int, C.c_uint, _f32p, _f32p, _szp]
        L.lr_evaluate.argtypes = [C.c_void_p, _f32p, _f32p, C.c_size_t, C.POINTER(C.c_float),
                                  C.POINTER(C.c_float)]
        L.lr_cross_entropy.restype = C.c_float
        L.lr_cross_entropy.argtypes = [_f32p, _f32p, C.c_size_t]
        L.lr_sgd_bench.restype = C.c_double
        L.lr_sgd_bench.argtypes = [C.c_void_p, _f32p, _f32p, C.c_size_t, C.c_void_p, C.c_size_t,
                                   C.c_size_t, C.c_float, C.c_int, C.c_uint, C.c_void_p]
        L.lr_net_hash.restype = C.c_uint64
        L.lr_net_hash.argtypes = [C.c_void_p]
        L.lr_rng_fill.argtypes = [C.c_uint64, C.c_size_t, C.c_float, C.c_float, _f32p]
        L.lr_rng_u64.argtypes = [C.c_uint64, C.c_size_t,
                                 np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")]
        L.lr_load_dataset.restype = C.c_long
        L.lr_load_dataset.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, _f32p, _f32p, C.c_size_t]
        L.lr_split.restype = C.c_long
        L.lr_split.argtypes = [_f32p, _f32p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_double,
                               C.c_uint64, _f32p, _f32p]
        L.lr_enlarge.argtypes = [_f32p, _f32p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.c_float, C.c_uint64, _f32p, _f32p]
        _ref = L
    return _ref


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _sizes(hidden):
    h = (C.c_size_t * max(1, len(hidden)))(*hidden)
    return h


class OracleNet:
    """The C restatement's FeedForwardNetwork (oracle/lane_oracle.c)."""

    def __init__(self, input_width, hidden, classes, seed=42, _ptr=None):
        L = oracle_lib()
        self.input_width, self.hidden, self.classes = input_width, list(hidden), classes
        self._p = _ptr if _ptr is not None else L.lo_net_new(
            input_width, _sizes(hidden), len(hidden), classes, seed)
        if not self._p:
            raise ValueError("oracle: bad topology")

    def __del__(self):
        if getattr(self, "_p", None):
            oracle_lib().lo_net_delete(self._p)
            self._p = None

    @property
    def n_layers(self):
        return len(self.hidden) + 1

    def clone(self):
        return OracleNet(self.input_width, self.hidden, self.classes,
                         _ptr=oracle_lib().lo_net_clone(self._p))

    def _view(self, layer, buf):
        n = C.c_size_t()
        p = oracle_lib().lo_net_buf(self._p, layer, buf, C.byref(n))
        if not p:
            raise IndexError((layer, buf))
        return np.ctypeslib.as_array(p, shape=(n.value,))

    def get(self, layer, buf):
        return self._view(layer, buf).copy()

    def set(self, layer, buf, values):
        v = self._view(layer, buf)
        v[:] = _f32(values).reshape(-1)

    def forward(self, x):
        p = oracle_lib().lo_net_forward(self._p, _f32(x))
        return np.ctypeslib.as_array(p, shape=(self.classes,)).copy()

    def backward_plan_run(self, t, eta):
        oracle_lib().lo_backward_plan_run(self._p, _f32(t), eta)

    def backward_no_update(self, t, eta):
        oracle_lib().lo_backward_no_update(self._p, _f32(t), eta)

    def train(self, X, T, eta, max_epochs=1, max_error=0.0, seed=0):
        st = (_Stats * max_epochs)()
        n = oracle_lib().lo_train(self._p, _f32(X), _f32(T), len(X), eta, max_error, max_epochs,
                                  seed, st)
        return [(st[e].epoch, st[e].mean_loss, st[e].accuracy) for e in range(n)]

    def evaluate(self, X, T):
        s = oracle_lib().lo_evaluate(self._p, _f32(X), _f32(T), len(X))
        return (s.mean_loss, s.accuracy)

    def sgd_run(self, X, T, n_steps, eta, order=None):
        o = None if order is None else np.ascontiguousarray(order, dtype=np.uint32)
        return oracle_lib().lo_sgd_run(self._p, _f32(X), _f32(T), len(X),
                                       None if o is None else o.ctypes.data, n_steps, eta)

    def minibatch_step(self, X, T, eta, mu):
        return oracle_lib().lo_minibatch_step(self._p, _f32(X), _f32(T), len(X), eta, mu)

    def hash(self):
        return int(oracle_lib().lo_net_hash(self._p))


class RefNet:
    """The reference's own lane::FeedForwardNetwork (oracle/_ref/liblane_ref.so)."""

    def __init__(self, input_width, hidden, classes, seed=42):
        L = ref_lib()
        self.input_width, self.hidden, self.classes = input_width, list(hidden), classes
        self._p = L.lr_net_create(input_width, _sizes(hidden), len(hidden), classes, seed)
        if not self._p:
            raise ValueError(L.lr_last_error().decode())

    def __del__(self):
        if getattr(self, "_p", None):
            ref_lib().lr_net_destroy(self._p)
            self._p = None

    @property
    def n_layers(self):
        return len(self.hidden) + 1

    def get(self, layer, buf):
        L = ref_lib()
        n = L.lr_net_rw(self._p, layer, buf, None, 0)
        out = np.empty(n, np.float32)
        L.lr_net_rw(self._p, layer, buf, out.ctypes.data, 0)
        return out

    def set(self, layer, buf, values):
        v = _f32(values).reshape(-1)
        ref_lib().lr_net_rw(self._p, layer, buf, v.ctypes.data, 1)

    def forward(self, x):
        p = np.empty(self.classes, np.float32)
        ref_lib().lr_net_forward(self._p, _f32(x), p)
        return p

    def backward_plan_run(self, t, eta, parallel=False, workers=0):
        tm = np.zeros(3 * self.n_layers, np.float64)
        rc = ref_lib().lr_backward_plan_run(self._p, _f32(t), eta, int(parallel), workers,
                                            tm.ctypes.data)
        if rc:
            raise RuntimeError(ref_lib().lr_last_error().decode())
        return tm

    def train(self, X, T, eta, max_epochs=1, max_error=0.0, seed=0, parallel=False, workers=0):
        loss = np.zeros(max_epochs, np.float32)
        acc = np.zeros(max_epochs, np.float32)
        n = C.c_size_t()
        rc = ref_lib().lr_train(self._p, _f32(X), _f32(T), len(X), eta, max_error, max_epochs,
                                seed, int(parallel), workers, loss, acc, C.byref(n))
        if rc:
            raise RuntimeError(ref_lib().lr_last_error().decode())
        return [(e + 1, float(loss[e]), float(acc[e])) for e in range(n.value)]

    def evaluate(self, X, T):
        lo, ac = C.c_float(), C.c_float()
        ref_lib().lr_evaluate(self._p, _f32(X), _f32(T), len(X), C.byref(lo), C.byref(ac))
        return (lo.value, ac.value)

    def sgd_bench(self, X, T, warmup, timed, eta, parallel=False, workers=0, order=None):
        ph = np.zeros(4, np.float64)
        o = None if order is None else np.ascontiguousarray(order, dtype=np.uint32)
        secs = ref_lib().lr_sgd_bench(self._p, _f32(X), _f32(T), len(X),
                                      None if o is None else o.ctypes.data, warmup, timed, eta,
                                      int(parallel), workers, ph.ctypes.data)
        if secs < 0:
            raise RuntimeError(ref_lib().lr_last_error().decode())
        return secs, ph

    def hash(self):
        return int(ref_lib().lr_net_hash(self._p))


# ------------------------------------------------------------ layer level --


def oracle_layer_backward(kind, outputs, inputs, eta, target=None, next_W=None, next_d=None):
    """Run lo_softmax_backward / lo_fc_backward on a standalone layer."""
    L = oracle_lib()
    outputs, inputs = _f32(outputs), _f32(inputs)
    I, O = inputs.size, outputs.size
    lp = L.lo_layer_new(I, O)
    lay = lp.contents
    np.ctypeslib.as_array(lay.a, shape=(O,))[:] = outputs
    np.ctypeslib.as_array(lay.x, shape=(I,))[:] = inputs
    if kind == "softmax":
        L.lo_softmax_backward(lp, _f32(target), eta)
    else:
        nW = _f32(next_W)
        L.lo_fc_backward(lp, nW.reshape(-1), nW.shape[1], _f32(next_d), eta)
    res = {
        "deltas": np.ctypeslib.as_array(lay.d, shape=(O,)).copy(),
        "gradients": np.ctypeslib.as_array(lay.G, shape=(I * O,)).copy().reshape(I, O),
        "delta_weights": np.ctypeslib.as_array(lay.DW, shape=(I * O,)).copy().reshape(I, O),
        "delta_biases": np.ctypeslib.as_array(lay.db, shape=(O,)).copy(),
    }
    L.lo_layer_delete(lp)
    return res


def oracle_layer_forward(kind, W, b, x):
    L = oracle_lib()
    W, b, x = _f32(W), _f32(b), _f32(x)
    I, O = W.shape
    lp = L.lo_layer_new(I, O)
    lay = lp.contents
    np.ctypeslib.as_array(lay.W, shape=(I * O,))[:] = W.reshape(-1)
    np.ctypeslib.as_array(lay.b, shape=(O,))[:] = b
    (L.lo_softmax_forward if kind == "softmax" else L.lo_fc_forward)(lp, x)
    z = np.ctypeslib.as_array(lay.z, shape=(O,)).copy()
    a = np.ctypeslib.as_array(lay.a, shape=(O,)).copy()
    L.lo_layer_delete(lp)
    return z, a


def ref_layer_backward(kind, outputs, inputs, eta, target=None, next_W=None, next_d=None):
    L = ref_lib()
    outputs, inputs = _f32(outputs), _f32(inputs)
    I, O = inputs.size, outputs.size
    d = np.zeros(O, np.float32)
    g = np.zeros(I * O, np.float32)
    dw = np.zeros(I * O, np.float32)
    db = np.zeros(O, np.float32)
    if kind == "softmax":
        t = _f32(target)
        rc = L.lr_softmax_backward(I, O, outputs, inputs, t, t.size, eta, d, g, dw, db)
    else:
        nW, nd = _f32(next_W), _f32(next_d)
        rc = L.lr_fc_backward(I, O, outputs, inputs, nW.shape[0], nW.shape[1], nW.reshape(-1),
                              nd, nd.size, eta, d, g, dw, db)
    if rc:
        raise RuntimeError(L.lr_last_error().decode())
    return {"deltas": d, "gradients": g.reshape(I, O), "delta_weights": dw.reshape(I, O),
            "delta_biases": db}


def ref_layer_forward(kind, W, b, x):
    L = ref_lib()
    W, b, x = _f32(W), _f32(b), _f32(x)
    I, O = W.shape
    z = np.zeros(O, np.float32)
    a = np.zeros(O, np.float32)
    rc = L.lr_layer_forward(int(kind == "softmax"), I, O, W.reshape(-1), b, x, z, a)
    if rc:
        raise RuntimeError(L.lr_last_error().decode())
    return z, a


# --------------------------------------------------------------- datasets --


def synthetic_dataset(features, classes, count, seed):
    """testsupport::synthetic_dataset (proj/tests/test_support.hpp:14-27)."""
    X = np.zeros((count, features), np.float32)
    T = np.zeros((count, classes), np.float32)
    oracle_lib().lo_synthetic_dataset(features, classes, count, seed, X.reshape(-1),
                                      T.reshape(-1))
    return X, T


def load_dataset(path, features, classes, cap=1 << 20):
    X = np.zeros((cap, features), np.float32) if cap < (1 << 16) else None
    # two-pass: count lines first to size the buffers
    with open(path) as f:
        n = sum(1 for line in f if line.strip())
    X = np.zeros((max(n, 1), features), np.float32)
    T = np.zeros((max(n, 1), classes), np.float32)
    got = oracle_lib().lo_load_dataset(path.encode(), features, classes, X.reshape(-1),
                                       T.reshape(-1), n)
    if got < 0:
        raise ValueError(f"cannot parse {path}")
    return X[:got], T[:got]


def split(X, T, frac, seed):
    """split (proj/src/dataset.cpp:103-124): returns (Xtr, Ttr, Xte, Tte)."""
    order = np.zeros(len(X), np.uint32)
    ntr = oracle_lib().lo_split_order(len(X), frac, seed, order)
    Xs, Ts = X[order], T[order]
    return Xs[:ntr], Ts[:ntr], Xs[ntr:], Ts[ntr:]


def shuffle_orders(n, epochs, seed):
    """The per-epoch sample orders train() visits (network.cpp:153-161): one
    SeededRng(seed), order not reset between epochs."""
    L = oracle_lib()
    rng = (C.c_uint64 * 2)()
    L.lo_rng_init(C.cast(rng, C.c_void_p), seed)
    order = np.arange(n, dtype=np.uint32)
    out = np.zeros((epochs, n), np.uint32)
    for e in range(epochs):
        for i in range(n, 1, -1):
            j = L.lo_rng_below(C.cast(rng, C.c_void_p), i)
            order[i - 1], order[j] = order[j], order[i - 1]
        out[e] = order
    return out
