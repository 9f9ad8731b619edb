"""Python mirror of the reference's ``lane`` layer/network API over the C ABI.

The reference API (``/root/reference/proj/include/lane/{layers,network}.hpp``)
is reproduced name for name -- ``LearningRate``, ``LayerState`` buffers,
``FullyConnectedLayer.forward/backward``, ``SoftmaxOutputLayer.forward/
backward``, ``apply_updates``, ``FeedForwardNetwork``, ``build_network``,
``BackwardPlan.run``, ``TrainerConfig``, ``EpochStats``, ``train``,
``evaluate`` -- with the same argument meaning and the same error types
(``ShapeError``, ``ConfigError``, ``TrainingError``, ... from
``include/lane/error.hpp``).  Every call goes through
``liblane_b200.so`` (``include/lane_b200.h``); state lives in HBM.  There is
no CPU fallback: importing this module on a machine without the built library
or without a B200 raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native

W, G, DW, B, INPUTS, NETIN, OUTPUTS, DELTAS, DELTA_BIASES, BIAS_GRAD = range(10)
NUMERICS_STRICT, NUMERICS_FAST = 0, 1


class Error(RuntimeError):
    """lane::Error (include/lane/error.hpp:8-10)."""


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class ScheduleError(Error):
    pass


class TrainingError(Error):
    pass


class IoError(Error):
    pass


class ParseError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


_ERRORS = {1: ShapeError, 2: ConfigError, 3: ScheduleError, 4: TrainingError, 5: IoError,
           6: ParseError, 7: CudaError, 8: NcclError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _native.lib().lane_b200_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


# --------------------------------------------------------------- device ---

class Device:
    """One GPU context (replaces lane::Device, task_runtime.hpp:97-127)."""

    def __init__(self, index: int = 0, numerics: int | None = None):
        L = _native.lib()
        self._p = C.c_void_p()
        _check(L.lane_b200_ctx_create(index, C.byref(self._p)))
        self.index = index
        self.world = 1
        if numerics is not None:
            self.numerics = numerics

    def close(self):
        if getattr(self, "_p", None) and self._p.value:
            _native.lib().lane_b200_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def numerics(self) -> int:
        m = C.c_int()
        _check(_native.lib().lane_b200_ctx_get_numerics(self._p, C.byref(m)))
        return m.value

    @numerics.setter
    def numerics(self, mode: int):
        _check(_native.lib().lane_b200_ctx_set_numerics(self._p, int(mode)))

    def sync(self):
        _check(_native.lib().lane_b200_sync(self._p))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(_native.lib().lane_b200_ctx_stream(self._p, C.byref(s)))
        return s.value or 0

    @property
    def kernel_launches(self) -> int:
        n = C.c_uint64()
        _check(_native.lib().lane_b200_kernel_launches(self._p, C.byref(n)))
        return n.value

    def alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        _check(_native.lib().lane_b200_dev_alloc(self._p, nbytes, C.byref(p)))
        return p.value

    def free(self, dev: int):
        _check(_native.lib().lane_b200_dev_free(self._p, C.c_void_p(dev)))

    def h2d(self, dev: int, host: np.ndarray):
        host = np.ascontiguousarray(host)
        _check(_native.lib().lane_b200_memcpy_h2d(self._p, C.c_void_p(dev), host.ctypes.data,
                                                  host.nbytes))

    def d2h(self, host: np.ndarray, dev: int):
        _check(_native.lib().lane_b200_memcpy_d2h(self._p, host.ctypes.data, C.c_void_p(dev),
                                                  host.nbytes))

    # data-parallel communicator (mini-batch extension)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_native.lib().lane_b200_nccl_unique_id(buf, 128))
        return buf.raw

    def comm_init(self, rank: int, world: int, uid: bytes):
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(_native.lib().lane_b200_comm_init(self._p, rank, world, buf, 128))
        self.world = int(world)

    def comm_destroy(self):
        _check(_native.lib().lane_b200_comm_destroy(self._p))
        self.world = 1

    def nvls_supported(self) -> bool:
        """Whether this GPU supports NVSwitch multicast objects (NVLS)."""
        v = C.c_int(0)
        _check(_native.lib().lane_b200_nvls_supported(self._p, C.byref(v)))
        return bool(v.value)


_default_device: Device | None = None


def default_device() -> Device:
    global _default_device
    if _default_device is None:
        _default_device = Device(int(os.environ.get("LANE_B200_DEVICE", "0")))
    return _default_device


# ---------------------------------------------------------------- layers ---

@dataclass(frozen=True)
class LearningRate:
    """layers.hpp:11-19: eta must be positive (ConfigError)."""
    eta: float

    def __post_init__(self):
        if not (self.eta > 0.0):
            raise ConfigError("LearningRate: eta must be positive")


def _eta(eta) -> float:
    return float(eta.eta if isinstance(eta, LearningRate) else LearningRate(float(eta)).eta)


class _Buffer:
    def __init__(self, name: int):
        self.id = name

    def __get__(self, layer, owner=None):
        if layer is None:
            return self
        return layer.read(self.id)

    def __set__(self, layer, value):
        layer.write(self.id, value)


class LayerState:
    """Device-resident LayerState (layers.hpp:68-92).  Buffer attributes read
    from / write to HBM; matrices come back as (cols_input, cols_out)."""

    weights = _Buffer(W)
    gradients = _Buffer(G)
    delta_weights = _Buffer(DW)
    biases = _Buffer(B)
    inputs = _Buffer(INPUTS)
    netin = _Buffer(NETIN)
    outputs = _Buffer(OUTPUTS)
    deltas = _Buffer(DELTAS)
    delta_biases = _Buffer(DELTA_BIASES)
    bias_gradients = _Buffer(BIAS_GRAD)

    def __init__(self, net: "FeedForwardNetwork", index: int):
        self._net, self.index = net, index
        ci, co = C.c_size_t(), C.c_size_t()
        _check(_native.lib().lane_b200_net_shape(net._p, index, C.byref(ci), C.byref(co)))
        self._in, self._out = ci.value, co.value

    def cols_input(self) -> int:
        return self._in

    def cols_out(self) -> int:
        return self._out

    def _count(self, buf):
        return {W: self._in * self._out, G: self._in * self._out, DW: self._in * self._out,
                INPUTS: self._in}.get(buf, self._out)

    def read(self, buf: int) -> np.ndarray:
        n = self._count(buf)
        out = np.empty(n, np.float32)
        _check(_native.lib().lane_b200_buf_read(self._net._p, self.index, buf, _ptr(out), n))
        return out.reshape(self._in, self._out) if buf in (W, G, DW) else out

    def write(self, buf: int, values) -> None:
        v = _f32(values).reshape(-1)
        if v.size != self._count(buf):
            raise ShapeError(f"buffer {buf}: expected {self._count(buf)} values, got {v.size}")
        _check(_native.lib().lane_b200_buf_write(self._net._p, self.index, buf, _ptr(v), v.size))

    def device_ptr(self, buf: int) -> int:
        p = C.POINTER(C.c_float)()
        _check(_native.lib().lane_b200_buf_device_ptr(self._net._p, self.index, buf, C.byref(p),
                                                      None))
        return C.cast(p, C.c_void_p).value

    def apply_updates(self) -> None:
        """weights += delta_weights; biases += delta_biases (layers.cpp:18-25)."""
        _check(_native.lib().lane_b200_apply_updates(self._net._p, self.index))

    def forward(self, x=None) -> np.ndarray:
        if x is None:
            rc = _native.lib().lane_b200_layer_forward(self._net._p, self.index, None, 0)
        else:
            x = _f32(x).reshape(-1)
            rc = _native.lib().lane_b200_layer_forward(self._net._p, self.index, _ptr(x), x.size)
        _check(rc)
        return self.outputs


class FullyConnectedLayer(LayerState):
    """layers.hpp:94-104: tanh FC layer."""

    def backward(self, next_weights=None, next_deltas=None, eta=0.01) -> None:
        """fc_backward_tuple over (o, i) (layers.cpp:51-69).  With no
        arguments, uses the next layer's device weights and deltas."""
        L = _native.lib()
        if next_weights is None:
            rc = L.lane_b200_fc_backward(self._net._p, self.index, None, 0, 0, None, 0, _eta(eta))
        else:
            nW = _f32(next_weights)
            if nW.ndim != 2:
                raise ShapeError("fc backward: next_weights must be a matrix")
            nd = _f32(next_deltas).reshape(-1)
            rc = L.lane_b200_fc_backward(self._net._p, self.index, _ptr(nW), nW.shape[0],
                                         nW.shape[1], _ptr(nd), nd.size, _eta(eta))
        _check(rc)


class SoftmaxOutputLayer(LayerState):
    """layers.hpp:106-114: softmax + one-hot cross-entropy output layer."""

    def backward(self, target, eta) -> None:
        t = _f32(target).reshape(-1)
        _check(_native.lib().lane_b200_softmax_backward(self._net._p, _ptr(t), t.size, _eta(eta)))


# --------------------------------------------------------------- network ---

class FeedForwardNetwork:
    """network.hpp:14-30.  Zero-initialised on construction (like the
    reference ctor); ``build_network`` adds the seeded initialisation."""

    def __init__(self, input_width: int, hidden_sizes, classes: int, device: Device | None = None,
                 max_batch: int = 1):
        self.device = device or default_device()
        hidden = [int(h) for h in hidden_sizes]
        arr = (C.c_size_t * max(1, len(hidden)))(*hidden)
        self._p = C.c_void_p()
        _check(_native.lib().lane_b200_net_create(self.device._p, int(input_width), arr,
                                                  len(hidden), int(classes), int(max_batch),
                                                  C.byref(self._p)))
        self._input_width, self.max_batch = int(input_width), int(max_batch)
        self.hidden = [FullyConnectedLayer(self, l) for l in range(len(hidden))]
        self.output = SoftmaxOutputLayer(self, len(hidden))

    def close(self):
        if getattr(self, "_p", None) and self._p.value:
            _native.lib().lane_b200_net_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def layers(self):
        return self.hidden + [self.output]

    def input_width(self) -> int:
        return self._input_width

    def class_count(self) -> int:
        return self.output.cols_out()

    def forward(self, x) -> np.ndarray:
        """FeedForwardNetwork::forward (network.cpp:47-53); returns probabilities."""
        x = _f32(x).reshape(-1)
        if x.size != self._input_width:
            raise ShapeError(f"forward: input length {x.size} != cols_input {self._input_width}")
        p = np.empty(self.class_count(), np.float32)
        _check(_native.lib().lane_b200_forward(self._p, _ptr(x), _ptr(p)))
        return p

    def init_seeded(self, seed: int) -> None:
        _check(_native.lib().lane_b200_net_init_seeded(self._p, C.c_uint64(seed)))

    def hash(self) -> int:
        """FNV-1a over weights and biases (bench.cpp:32-41)."""
        h = C.c_uint64()
        _check(_native.lib().lane_b200_net_hash(self._p, C.byref(h)))
        return h.value

    # -- fused online SGD over a device-resident stream ------------------
    def sgd_stream(self, X_dev: int, T_dev: int, n: int, n_steps: int, eta, order_dev: int = 0,
                   loss_dev: int = 0, correct_dev: int = 0) -> None:
        _check(_native.lib().lane_b200_sgd_stream(
            self._p, C.c_void_p(X_dev), C.c_void_p(T_dev), n, C.c_void_p(order_dev or None),
            n_steps, C.c_float(_eta(eta)), C.c_void_p(loss_dev or None),
            C.c_void_p(correct_dev or None)))

    def sgd_plan(self) -> str:
        """The fused plan sgd_stream runs for this network ("window ...",
        "cluster ...", "grid ..." or "layer")."""
        buf = C.create_string_buffer(128)
        _check(_native.lib().lane_b200_sgd_stream_plan(self._p, buf, 128))
        return buf.value.decode()

    # -- mini-batch extension --------------------------------------------
    def minibatch_step(self, X_dev: int, T_dev: int, batch: int, eta, mu: float = 0.0,
                       loss_dev: int = 0) -> None:
        _check(_native.lib().lane_b200_minibatch_step(
            self._p, C.c_void_p(X_dev), C.c_void_p(T_dev), batch, C.c_float(_eta(eta)),
            C.c_float(mu), C.c_void_p(loss_dev or None)))

    def minibatch_grads(self, X_dev: int, T_dev: int, batch: int, loss_dev: int = 0) -> None:
        """Forward + backward of a device batch: gradient sums into the grads
        arena, no update (lane_b200_minibatch_grads)."""
        _check(_native.lib().lane_b200_minibatch_grads(
            self._p, C.c_void_p(X_dev), C.c_void_p(T_dev), batch, C.c_void_p(loss_dev or None)))

    def minibatch_apply(self, global_batch: int, eta, mu: float = 0.0) -> None:
        """The update from the arena's gradient sums (lane_b200_minibatch_apply)."""
        _check(_native.lib().lane_b200_minibatch_apply(self._p, global_batch, C.c_float(_eta(eta)),
                                                       C.c_float(mu)))

    def grads_arena(self) -> tuple[int, int]:
        """(device pointer, float count) of the flat gradient arena."""
        p, n = C.c_void_p(), C.c_size_t()
        _check(_native.lib().lane_b200_net_grads_arena(self._p, C.byref(p), C.byref(n)))
        return p.value, n.value

    def allreduce_grads(self) -> None:
        _check(_native.lib().lane_b200_allreduce_grads(self._p))

    # NVLS fused exchange + update (csrc/nvls.cuh); parallel.init_nvls drives
    # the multi-rank sequence
    def nvls_create(self, world: int, export: bool = True) -> int:
        fd = C.c_int(-1)
        _check(_native.lib().lane_b200_nvls_create(self._p, world, C.byref(fd) if export else None))
        return fd.value

    def nvls_attach(self, rank: int, world: int, fd: int = -1) -> None:
        _check(_native.lib().lane_b200_nvls_attach(self._p, rank, world, fd))

    def nvls_bind(self) -> None:
        _check(_native.lib().lane_b200_nvls_bind(self._p))

    def nvls_mode(self) -> str:
        """"multicast", "local" (one rank without a multicast object) or "off"."""
        v = C.c_int(-1)
        _check(_native.lib().lane_b200_nvls_mode(self._p, C.byref(v)))
        return {1: "multicast", 0: "local"}.get(v.value, "off")


def build_network(input_width: int, hidden_sizes, classes: int, seed: int = 42,
                  device: Device | None = None, max_batch: int = 1) -> FeedForwardNetwork:
    """build_network (network.cpp:55-66) with SeededRng(seed): bit-identical
    initial weights to the reference."""
    net = FeedForwardNetwork(input_width, hidden_sizes, classes, device, max_batch)
    net.init_seeded(seed)
    return net


class BackwardPlan:
    """network.hpp:58-75.  ``run(target)``: output backward, hidden backward in
    reverse, then apply_updates on every layer (network.cpp:122-138)."""

    def __init__(self, net: FeedForwardNetwork, eta):
        self.net, self.eta = net, _eta(eta)

    def run(self, target) -> None:
        t = _f32(target).reshape(-1)
        if t.size != self.net.class_count():
            raise ShapeError("backward: target length != class count")
        _check(_native.lib().lane_b200_backward_plan_run(self.net._p, _ptr(t), self.eta))

    def run_timed(self, target) -> list["PhaseTiming"]:
        """run() returning one PhaseTiming per schedule, output layer first
        (network.hpp:70-72); device-timed with CUDA events, blocking."""
        t = _f32(target).reshape(-1)
        if t.size != self.net.class_count():
            raise ShapeError("backward: target length != class count")
        nl = len(self.net.layers)
        ph = (C.c_double * (3 * nl))()
        _check(_native.lib().lane_b200_backward_plan_run_timed(self.net._p, _ptr(t), self.eta, ph, 3 * nl))
        return [PhaseTiming(ph[3 * k], ph[3 * k + 1], ph[3 * k + 2]) for k in range(nl)]


@dataclass
class PhaseTiming:
    """task_runtime.hpp:53-60 (milliseconds)."""
    copy_in_ms: float = 0.0
    kernel_ms: float = 0.0
    copy_out_ms: float = 0.0

    def total_ms(self) -> float:
        return self.copy_in_ms + self.kernel_ms + self.copy_out_ms


@dataclass
class TrainerConfig:
    """network.hpp:41-46."""
    eta: LearningRate = LearningRate(0.01)
    max_error: float = 0.0
    max_epochs: int = 1
    seed: int = 0


@dataclass
class EpochStats:
    """network.hpp:48-52."""
    epoch: int = 0
    mean_loss: float = 0.0
    accuracy: float = 0.0


@dataclass
class DataSet:
    """dataset.hpp:16-23: features (n x feature_width), labels one-hot (n x
    classes).  Sets made by load_dataset / split / enlarge are views of the
    library's page-locked rows (``_owner`` keeps them alive)."""
    features: np.ndarray
    labels: np.ndarray
    _owner: object = field(default=None, repr=False, compare=False)

    @property
    def feature_width(self) -> int:
        return int(self.features.shape[1])

    @property
    def class_count(self) -> int:
        return int(self.labels.shape[1])

    def size(self) -> int:
        return int(self.features.shape[0])


def _check_set(net: FeedForwardNetwork, d: DataSet, what: str) -> None:
    if d.size() == 0:
        raise TrainingError(f"{what}: empty {'training' if what == 'train' else 'test'} set")
    if d.feature_width != net.input_width():
        raise ShapeError(f"{what}: dataset feature width != network input width")
    if d.class_count != net.class_count():
        raise ShapeError(f"{what}: dataset class count != network class count")


def train(net: FeedForwardNetwork, train_set: DataSet, cfg: TrainerConfig) -> list[EpochStats]:
    """train (network.cpp:140-182): seed-deterministic shuffle per epoch, fused
    online SGD on the GPU, early stop on max_error."""
    _check_set(net, train_set, "train")
    n, E = train_set.size(), int(cfg.max_epochs)
    loss = np.zeros(max(1, E), np.float32)
    acc = np.zeros(max(1, E), np.float32)
    ran = C.c_size_t()
    X, T = _f32(train_set.features), _f32(train_set.labels)
    _check(_native.lib().lane_b200_train(net._p, _ptr(X), _ptr(T), n, C.c_float(_eta(cfg.eta)),
                                         C.c_float(cfg.max_error), E, C.c_uint64(cfg.seed),
                                         _ptr(loss), _ptr(acc), C.byref(ran)))
    return [EpochStats(e + 1, float(loss[e]), float(acc[e])) for e in range(ran.value)]


def evaluate(net: FeedForwardNetwork, test_set: DataSet) -> EpochStats:
    """evaluate (network.cpp:184-204)."""
    _check_set(net, test_set, "evaluate")
    X, T = _f32(test_set.features), _f32(test_set.labels)
    lo, ac = C.c_float(), C.c_float()
    _check(_native.lib().lane_b200_evaluate(net._p, _ptr(X), _ptr(T), test_set.size(),
                                            C.byref(lo), C.byref(ac)))
    return EpochStats(0, lo.value, ac.value)


# ------------------------------------------------------------------ datasets
class _NativeSet:
    """Owns a lane_b200_dataset handle (page-locked rows)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _native.lib().lane_b200_dataset_destroy(h)


def _wrap_native(handle) -> DataSet:
    L = _native.lib()
    F, Cn, n = C.c_size_t(), C.c_size_t(), C.c_size_t()
    xp, tp = C.POINTER(C.c_float)(), C.POINTER(C.c_float)()
    pinned = C.c_int()
    _check(L.lane_b200_dataset_info(handle, C.byref(F), C.byref(Cn), C.byref(n), C.byref(xp), C.byref(tp),
                                    C.byref(pinned)))
    owner = _NativeSet(handle)
    if n.value == 0:
        return DataSet(np.zeros((0, F.value), np.float32), np.zeros((0, Cn.value), np.float32), owner)
    X = np.ctypeslib.as_array(xp, shape=(n.value, F.value))
    T = np.ctypeslib.as_array(tp, shape=(n.value, Cn.value))
    return DataSet(X, T, owner)


def _to_native(d: DataSet):
    """A native handle for d (reuses d's own when it has one)."""
    if isinstance(d._owner, _NativeSet):
        return d._owner._h, None
    X, T = _f32(d.features), _f32(d.labels)
    h = C.c_void_p()
    _check(_native.lib().lane_b200_dataset_create(X.shape[1], T.shape[1], X.shape[0], _ptr(X), _ptr(T),
                                                  C.byref(h)))
    tmp = _NativeSet(h)
    return h, tmp


class SeededRng:
    """SplitMix64 state (tensor.hpp:13-44) for enlarge(); advanced in place."""

    def __init__(self, seed: int = 0):
        self.state = int(seed) & 0xFFFFFFFFFFFFFFFF


def load_dataset(path, feature_width: int, class_count: int) -> DataSet:
    """load_dataset (dataset.hpp:25-30, dataset.cpp:31-83)."""
    h = C.c_void_p()
    _check(_native.lib().lane_b200_dataset_load(os.fsencode(path), feature_width, class_count, C.byref(h)))
    return _wrap_native(h)


def save_dataset(d: DataSet, path) -> None:
    """save_dataset (dataset.hpp:32-33, dataset.cpp:85-103)."""
    h, _tmp = _to_native(d)
    _check(_native.lib().lane_b200_dataset_save(h, os.fsencode(path)))


def split(d: DataSet, train_fraction: float, seed: int) -> tuple[DataSet, DataSet]:
    """split (dataset.hpp:35-37, dataset.cpp:105-124)."""
    h, _tmp = _to_native(d)
    a, b = C.c_void_p(), C.c_void_p()
    _check(_native.lib().lane_b200_dataset_split(h, float(train_fraction), C.c_uint64(seed), C.byref(a),
                                                 C.byref(b)))
    return _wrap_native(a), _wrap_native(b)


def enlarge(d: DataSet, factor: int, noise: float, rng: SeededRng) -> DataSet:
    """enlarge (dataset.hpp:39-41, dataset.cpp:126-148)."""
    if factor < 0:
        raise ConfigError("enlarge: factor must be >= 1")
    h, _tmp = _to_native(d)
    st = C.c_uint64(rng.state)
    out = C.c_void_p()
    _check(_native.lib().lane_b200_dataset_enlarge(h, factor, C.c_float(noise), C.byref(st), C.byref(out)))
    rng.state = st.value
    return _wrap_native(out)


def train_minibatch(net: FeedForwardNetwork, train_set: DataSet, batch: int, eta, mu: float = 0.0,
                    epochs: int = 1, seed: int = 0, shuffle: bool = True, drop_last: bool = True,
                    step_losses: bool = False):
    """Mini-batch training over a host dataset through the pipelined input
    path (lane_b200_train_minibatch).  Returns the per-epoch mean losses, and
    with step_losses=True also the per-step mean losses [epochs, steps]."""
    _check_set(net, train_set, "train")
    X, T = _f32(train_set.features), _f32(train_set.labels)
    n = train_set.size()
    world = getattr(net.device, "world", 1)
    bg = batch * world
    steps = n // bg + (1 if (world == 1 and not drop_last and n % bg) else 0)
    E = int(epochs)
    ml = np.zeros(max(1, E), np.float32)
    sl = np.zeros(max(1, E * max(1, steps)), np.float32) if step_losses else None
    ran = C.c_size_t()
    _check(_native.lib().lane_b200_train_minibatch(
        net._p, _ptr(X), _ptr(T), n, batch, C.c_float(_eta(eta)), C.c_float(mu), E, C.c_uint64(seed),
        int(bool(shuffle)), int(bool(drop_last)), _ptr(ml), _ptr(sl) if sl is not None else None,
        C.byref(ran)))
    if step_losses:
        return [float(v) for v in ml[:E]], sl[:E * steps].reshape(E, steps)
    return [float(v) for v in ml[:E]]
