// lane_b200/lane.hpp -- C++ facade over the C ABI (include/lane_b200.h) that
// restores the reference's layer/network API (namespace lane, proj/include/
// lane/{error,layers,network}.hpp) on B200-resident state.  Header-only; link
// against paper_2001_04206_b200/lib/liblane_b200.so.
//
//   reference                                   here
//   lane::Device(Kind, workers)                 lane_b200::Device(gpu)
//   lane::build_network(in, hidden, C, rng)     lane_b200::build_network(dev, in, hidden, C, seed)
//   FullyConnectedLayer::forward / backward     same names (device buffers behind them)
//   SoftmaxOutputLayer::forward / backward      same names
//   LayerState::apply_updates                   same name
//   BackwardPlan(net, eta, dev).run(target)     BackwardPlan(net, eta).run(target)
//   train(net, set, cfg, dev) / evaluate        train(net, set, cfg) / evaluate(net, set)
//   lane::ShapeError, ConfigError, ...          lane_b200::ShapeError, ConfigError, ...
//
// Buffers are read/written through LayerState::read()/write() (host vectors),
// the device-resident analogue of the reference's public std::vector members.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../lane_b200.h"

namespace lane_b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct ScheduleError : Error {
    using Error::Error;
};
struct TrainingError : Error {
    using Error::Error;
};
struct IoError : Error {
    using Error::Error;
};
struct ParseError : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == LANE_OK) return;
    const std::string msg = lane_b200_last_error();
    switch (rc) {
        case LANE_ERR_SHAPE: throw ShapeError(msg);
        case LANE_ERR_CONFIG: throw ConfigError(msg);
        case LANE_ERR_SCHEDULE: throw ScheduleError(msg);
        case LANE_ERR_TRAINING: throw TrainingError(msg);
        case LANE_ERR_IO: throw IoError(msg);
        case LANE_ERR_PARSE: throw ParseError(msg);
        default: throw DeviceError(msg);
    }
}

// layers.hpp:11-19
struct LearningRate {
    float eta;
    explicit LearningRate(float e) : eta(e) {
        if (!(eta > 0.0f)) throw ConfigError("LearningRate: eta must be positive");
    }
};

enum class Numerics { Strict = LANE_NUMERICS_STRICT, Fast = LANE_NUMERICS_FAST };

class Device {
public:
    explicit Device(int gpu = 0, Numerics mode = Numerics::Fast) {
        check(lane_b200_ctx_create(gpu, &ctx_));
        check(lane_b200_ctx_set_numerics(ctx_, static_cast<int>(mode)));
    }
    ~Device() { lane_b200_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    void set_numerics(Numerics m) { check(lane_b200_ctx_set_numerics(ctx_, static_cast<int>(m))); }
    void sync() { check(lane_b200_sync(ctx_)); }
    lane_b200_ctx* handle() const { return ctx_; }

private:
    lane_b200_ctx* ctx_ = nullptr;
};

class FeedForwardNetwork;

// layers.hpp:68-92 -- the buffers live in HBM; read()/write() copy them.
class LayerState {
public:
    std::size_t cols_input() const { return in_; }
    std::size_t cols_out() const { return out_; }
    std::vector<float> read(int buf) const {
        std::vector<float> v(count(buf));
        check(lane_b200_buf_read(net_, index_, buf, v.data(), v.size()));
        return v;
    }
    void write(int buf, const std::vector<float>& v) {
        if (v.size() != count(buf)) throw ShapeError("LayerState::write: size mismatch");
        check(lane_b200_buf_write(net_, index_, buf, v.data(), v.size()));
    }
    std::vector<float> weights() const { return read(LANE_BUF_W); }
    std::vector<float> gradients() const { return read(LANE_BUF_G); }
    std::vector<float> delta_weights() const { return read(LANE_BUF_DW); }
    std::vector<float> biases() const { return read(LANE_BUF_B); }
    std::vector<float> inputs() const { return read(LANE_BUF_INPUTS); }
    std::vector<float> netin() const { return read(LANE_BUF_NETIN); }
    std::vector<float> outputs() const { return read(LANE_BUF_OUTPUTS); }
    std::vector<float> deltas() const { return read(LANE_BUF_DELTAS); }
    std::vector<float> delta_biases() const { return read(LANE_BUF_DELTA_BIASES); }

    // layers.cpp:18-25
    void apply_updates() { check(lane_b200_apply_updates(net_, index_)); }

    // layers.cpp:27-49 / :71-87
    std::vector<float> forward(const std::vector<float>& input) {
        check(lane_b200_layer_forward(net_, index_, input.data(), input.size()));
        return outputs();
    }

protected:
    friend class FeedForwardNetwork;
    LayerState(lane_b200_net* net, std::size_t index) : net_(net), index_(index) {
        check(lane_b200_net_shape(net, index, &in_, &out_));
    }
    std::size_t count(int buf) const {
        return (buf == LANE_BUF_W || buf == LANE_BUF_G || buf == LANE_BUF_DW) ? in_ * out_
               : buf == LANE_BUF_INPUTS                                       ? in_
                                                                              : out_;
    }
    lane_b200_net* net_;
    std::size_t index_, in_ = 0, out_ = 0;
};

struct FullyConnectedLayer : LayerState {
    // layers.cpp:51-69: next_weights is cols_out x next_cols_out, row-major
    void backward(const std::vector<float>& next_weights, std::size_t next_rows,
                  std::size_t next_cols, const std::vector<float>& next_deltas, LearningRate eta) {
        if (next_weights.size() != next_rows * next_cols)
            throw ShapeError("fc backward: next_weights storage != rows*cols");
        check(lane_b200_fc_backward(net_, index_, next_weights.data(), next_rows, next_cols,
                                    next_deltas.data(), next_deltas.size(), eta.eta));
    }
    // in-network form: uses the next layer's device weights and deltas
    void backward(LearningRate eta) {
        check(lane_b200_fc_backward(net_, index_, nullptr, 0, 0, nullptr, 0, eta.eta));
    }

private:
    friend class FeedForwardNetwork;
    FullyConnectedLayer(lane_b200_net* n, std::size_t i) : LayerState(n, i) {}
};

struct SoftmaxOutputLayer : LayerState {
    // layers.cpp:89-102
    void backward(const std::vector<float>& target, LearningRate eta) {
        check(lane_b200_softmax_backward(net_, target.data(), target.size(), eta.eta));
    }

private:
    friend class FeedForwardNetwork;
    SoftmaxOutputLayer(lane_b200_net* n, std::size_t i) : LayerState(n, i) {}
};

struct EpochStats {
    std::size_t epoch = 0;
    float mean_loss = 0.0f;
    float accuracy = 0.0f;
};

struct TrainerConfig {
    LearningRate eta{0.01f};
    float max_error = 0.0f;
    std::size_t max_epochs = 1;
    std::uint64_t seed = 0;
};

// features: n x feature_width, labels: n x classes (one-hot), row-major
struct DataSet {
    std::size_t feature_width = 0, class_count = 0;
    std::vector<float> features, labels;
    std::size_t size() const { return feature_width ? features.size() / feature_width : 0; }
};

// network.hpp:14-30
class FeedForwardNetwork {
public:
    FeedForwardNetwork(Device& dev, std::size_t input_width, const std::vector<std::size_t>& hidden,
                       std::size_t classes, std::size_t max_batch = 1)
        : input_width_(input_width) {
        check(lane_b200_net_create(dev.handle(), input_width, hidden.data(), hidden.size(), classes,
                                   max_batch, &net_));
        for (std::size_t l = 0; l < hidden.size(); ++l) this->hidden.push_back(FullyConnectedLayer(net_, l));
        output_.reset(new SoftmaxOutputLayer(net_, hidden.size()));
    }
    ~FeedForwardNetwork() { lane_b200_net_destroy(net_); }
    FeedForwardNetwork(const FeedForwardNetwork&) = delete;
    FeedForwardNetwork& operator=(const FeedForwardNetwork&) = delete;

    std::size_t input_width() const { return input_width_; }
    std::size_t class_count() const { return output_->cols_out(); }
    SoftmaxOutputLayer& output() { return *output_; }

    // network.cpp:47-53
    std::vector<float> forward(const std::vector<float>& input) {
        if (input.size() != input_width_) throw ShapeError("forward: input length != cols_input");
        std::vector<float> p(class_count());
        check(lane_b200_forward(net_, input.data(), p.data()));
        return p;
    }
    void init_seeded(std::uint64_t seed) { check(lane_b200_net_init_seeded(net_, seed)); }
    std::uint64_t hash() const {
        std::uint64_t h = 0;
        check(lane_b200_net_hash(net_, &h));
        return h;
    }
    lane_b200_net* handle() const { return net_; }

    std::vector<FullyConnectedLayer> hidden;

private:
    lane_b200_net* net_ = nullptr;
    std::size_t input_width_;
    std::unique_ptr<SoftmaxOutputLayer> output_;
};

// network.cpp:55-66 with SeededRng(seed)
inline std::unique_ptr<FeedForwardNetwork> build_network(Device& dev, std::size_t input_width,
                                                         const std::vector<std::size_t>& hidden,
                                                         std::size_t classes, std::uint64_t seed,
                                                         std::size_t max_batch = 1) {
    auto net = std::make_unique<FeedForwardNetwork>(dev, input_width, hidden, classes, max_batch);
    net->init_seeded(seed);
    return net;
}

// task_runtime.hpp:53-60
struct PhaseTiming {
    double copy_in_ms = 0.0;
    double kernel_ms = 0.0;
    double copy_out_ms = 0.0;
    double total_ms() const { return copy_in_ms + kernel_ms + copy_out_ms; }
};

// network.hpp:58-75
class BackwardPlan {
public:
    BackwardPlan(FeedForwardNetwork& net, LearningRate eta) : net_(net), eta_(eta) {}
    // Blocking, like the reference: one PhaseTiming per schedule, output first.
    std::vector<PhaseTiming> run(const std::vector<float>& target) {
        if (target.size() != net_.class_count()) throw ShapeError("backward: target length != class count");
        const std::size_t nl = net_.hidden.size() + 1;
        std::vector<double> ph(3 * nl);
        check(lane_b200_backward_plan_run_timed(net_.handle(), target.data(), eta_.eta, ph.data(), ph.size()));
        std::vector<PhaseTiming> out(nl);
        for (std::size_t k = 0; k < nl; ++k) out[k] = {ph[3 * k], ph[3 * k + 1], ph[3 * k + 2]};
        return out;
    }
    // Stream-ordered (no host sync, no timings): the production path.
    void run_async(const std::vector<float>& target) {
        if (target.size() != net_.class_count()) throw ShapeError("backward: target length != class count");
        check(lane_b200_backward_plan_run(net_.handle(), target.data(), eta_.eta));
    }

private:
    FeedForwardNetwork& net_;
    LearningRate eta_;
};

// network.cpp:140-182
inline std::vector<EpochStats> train(FeedForwardNetwork& net, const DataSet& set, const TrainerConfig& cfg) {
    if (set.size() == 0) throw TrainingError("train: empty training set");
    if (set.feature_width != net.input_width()) throw ShapeError("train: dataset feature width != network input width");
    if (set.class_count != net.class_count()) throw ShapeError("train: dataset class count != network class count");
    std::vector<float> loss(cfg.max_epochs), acc(cfg.max_epochs);
    std::size_t ran = 0;
    check(lane_b200_train(net.handle(), set.features.data(), set.labels.data(), set.size(), cfg.eta.eta,
                          cfg.max_error, cfg.max_epochs, cfg.seed, loss.data(), acc.data(), &ran));
    std::vector<EpochStats> out;
    for (std::size_t e = 0; e < ran; ++e) out.push_back({e + 1, loss[e], acc[e]});
    return out;
}

// network.cpp:184-204
inline EpochStats evaluate(FeedForwardNetwork& net, const DataSet& set) {
    if (set.size() == 0) throw TrainingError("evaluate: empty test set");
    if (set.feature_width != net.input_width() || set.class_count != net.class_count())
        throw ShapeError("evaluate: dataset shape does not match network");
    EpochStats es;
    check(lane_b200_evaluate(net.handle(), set.features.data(), set.labels.data(), set.size(), &es.mean_loss,
                             &es.accuracy));
    return es;
}

// ---------------------------------------------------------------- datasets
// dataset.hpp:25-41 over the library's loader (csrc/dataset.cuh); the
// library's page-locked rows are copied into the value-type DataSet.
struct SeededRng {  // tensor.hpp:13-44, only the state crosses the ABI
    std::uint64_t state;
    explicit SeededRng(std::uint64_t seed) : state(seed) {}
};

namespace detail {
struct NativeSet {
    lane_b200_dataset* h = nullptr;
    ~NativeSet() { lane_b200_dataset_destroy(h); }
    DataSet take() const {
        std::size_t F = 0, C = 0, n = 0;
        float *X = nullptr, *T = nullptr;
        check(lane_b200_dataset_info(h, &F, &C, &n, &X, &T, nullptr));
        DataSet d;
        d.feature_width = F;
        d.class_count = C;
        d.features.assign(X, X + n * F);
        d.labels.assign(T, T + n * C);
        return d;
    }
};
inline NativeSet to_native(const DataSet& d) {
    NativeSet s;
    check(lane_b200_dataset_create(d.feature_width, d.class_count, d.size(), d.features.data(), d.labels.data(),
                                   &s.h));
    return s;
}
}  // namespace detail

inline DataSet load_dataset(const std::string& path, std::size_t feature_width, std::size_t class_count) {
    detail::NativeSet s;
    check(lane_b200_dataset_load(path.c_str(), feature_width, class_count, &s.h));
    return s.take();
}

inline void save_dataset(const DataSet& d, const std::string& path) {
    check(lane_b200_dataset_save(detail::to_native(d).h, path.c_str()));
}

inline std::pair<DataSet, DataSet> split(const DataSet& d, double train_fraction, std::uint64_t seed) {
    detail::NativeSet a, b;
    check(lane_b200_dataset_split(detail::to_native(d).h, train_fraction, seed, &a.h, &b.h));
    return {a.take(), b.take()};
}

inline DataSet enlarge(const DataSet& d, std::size_t factor, float noise, SeededRng& rng) {
    detail::NativeSet e;
    check(lane_b200_dataset_enlarge(detail::to_native(d).h, factor, noise, &rng.state, &e.h));
    return e.take();
}

// Mini-batch extension over a host dataset with the pipelined input path
// (lane_b200_train_minibatch); returns the per-epoch mean losses.
inline std::vector<float> train_minibatch(FeedForwardNetwork& net, const DataSet& set, std::size_t batch,
                                          LearningRate eta, float momentum, std::size_t epochs,
                                          std::uint64_t seed, bool shuffle = true, bool drop_last = true) {
    if (set.size() == 0) throw TrainingError("train: empty training set");
    if (set.feature_width != net.input_width()) throw ShapeError("train: dataset feature width != network input width");
    if (set.class_count != net.class_count()) throw ShapeError("train: dataset class count != network class count");
    std::vector<float> loss(epochs);
    check(lane_b200_train_minibatch(net.handle(), set.features.data(), set.labels.data(), set.size(), batch,
                                    eta.eta, momentum, epochs, seed, shuffle ? 1 : 0, drop_last ? 1 : 0,
                                    loss.data(), nullptr, nullptr));
    return loss;
}

}  // namespace lane_b200
