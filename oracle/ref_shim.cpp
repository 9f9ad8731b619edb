// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources (/root/reference/proj/src/*.cpp, read in place,
// never copied) into oracle/_ref/liblane_ref.so.  Every entry point calls the
// reference's public API (lane::build_network, FeedForwardNetwork::forward,
// BackwardPlan::run, train, evaluate, the layer backward methods,
// load_dataset/split/enlarge); nothing here re-implements an algorithm.  It is
// used (a) to pin oracle/lane_oracle.c bit-for-bit, (b) to generate
// tests/golden/, and (c) as bench.py's "reference" CPU arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "lane/bench.hpp"
#include "lane/dataset.hpp"
#include "lane/network.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const lane::ShapeError*>(&e)) return 1;
    if (dynamic_cast<const lane::ConfigError*>(&e)) return 2;
    if (dynamic_cast<const lane::ScheduleError*>(&e)) return 3;
    if (dynamic_cast<const lane::TrainingError*>(&e)) return 4;
    if (dynamic_cast<const lane::IoError*>(&e)) return 5;
    if (dynamic_cast<const lane::ParseError*>(&e)) return 6;
    return 9;
}

lane::LayerState& layer_of(lane::FeedForwardNetwork& net, std::size_t l) {
    if (l < net.hidden.size()) return net.hidden[l];
    return net.output;
}

std::vector<float>* buf_of(lane::LayerState& L, int buf) {
    switch (buf) {
        case 0: return &L.weights.data;
        case 1: return &L.gradients.data;
        case 2: return &L.delta_weights.data;
        case 3: return &L.biases.data;
        case 4: return &L.inputs.data;
        case 5: return &L.netin.data;
        case 6: return &L.outputs.data;
        case 7: return &L.deltas.data;
        case 8: return &L.delta_biases.data;
        default: return nullptr;
    }
}

lane::DenseVector vec(const float* p, std::size_t n) {
    lane::DenseVector v(n);
    std::memcpy(v.data.data(), p, n * sizeof(float));
    return v;
}

lane::DataSet make_set(const float* X, const float* T, std::size_t n, std::size_t F,
                       std::size_t C) {
    lane::DataSet d;
    d.feature_width = F;
    d.class_count = C;
    d.items.reserve(n);
    for (std::size_t k = 0; k < n; ++k) d.items.push_back({vec(X + k * F, F), vec(T + k * C, C)});
    return d;
}

lane::Device::Kind kind_of(int parallel) {
    return parallel ? lane::Device::Kind::ParallelHost : lane::Device::Kind::SerialHost;
}

}  // namespace

extern "C" {

const char* lr_last_error() { return g_err.c_str(); }

void* lr_net_create(std::size_t in, const std::size_t* hidden, std::size_t nh, std::size_t classes,
                    std::uint64_t seed) {
    try {
        lane::SeededRng rng(seed);
        std::vector<std::size_t> h(hidden, hidden + nh);
        return new lane::FeedForwardNetwork(lane::build_network(in, h, classes, rng));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void lr_net_destroy(void* net) { delete static_cast<lane::FeedForwardNetwork*>(net); }

// Copies a LayerState buffer out (write == 0) or in (write != 0).  Returns the
// element count, or -1 for a bad layer/buffer id.
long lr_net_rw(void* netp, std::size_t layer, int buf, float* data, int write) {
    auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
    if (layer > net.hidden.size()) return -1;
    std::vector<float>* b = buf_of(layer_of(net, layer), buf);
    if (!b) return -1;
    if (data) {
        if (write) std::memcpy(b->data(), data, b->size() * sizeof(float));
        else std::memcpy(data, b->data(), b->size() * sizeof(float));
    }
    return static_cast<long>(b->size());
}

int lr_net_forward(void* netp, const float* x, float* p_out) {
    try {
        auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
        const lane::DenseVector& p = net.forward(vec(x, net.input_width()));
        if (p_out) std::memcpy(p_out, p.data.data(), p.len() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// BackwardPlan(net, eta, device).run(target); timings: per layer, output first,
// (copy_in, kernel, copy_out) ms.
int lr_backward_plan_run(void* netp, const float* t, float eta, int parallel, unsigned workers,
                         double* timings) {
    try {
        auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
        lane::Device dev(kind_of(parallel), workers);
        lane::BackwardPlan plan(net, lane::LearningRate(eta), dev);
        auto ts = plan.run(vec(t, net.class_count()));
        if (timings)
            for (std::size_t k = 0; k < ts.size(); ++k) {
                timings[3 * k] = ts[k].copy_in_ms;
                timings[3 * k + 1] = ts[k].kernel_ms;
                timings[3 * k + 2] = ts[k].copy_out_ms;
            }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Layer-level backward methods on standalone layers (test_layers.cpp style):
// the caller supplies outputs/inputs (and next-layer weights/deltas), the
// reference writes deltas, gradients, delta_weights, delta_biases.
int lr_softmax_backward(std::size_t in, std::size_t out, const float* outputs, const float* inputs,
                        const float* target, std::size_t target_len, float eta, float* deltas,
                        float* G, float* DW, float* db) {
    try {
        lane::SoftmaxOutputLayer L(in, out);
        std::memcpy(L.outputs.data.data(), outputs, out * sizeof(float));
        std::memcpy(L.inputs.data.data(), inputs, in * sizeof(float));
        L.backward(vec(target, target_len), lane::LearningRate(eta));
        std::memcpy(deltas, L.deltas.data.data(), out * sizeof(float));
        std::memcpy(G, L.gradients.data.data(), in * out * sizeof(float));
        std::memcpy(DW, L.delta_weights.data.data(), in * out * sizeof(float));
        std::memcpy(db, L.delta_biases.data.data(), out * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int lr_fc_backward(std::size_t in, std::size_t out, const float* outputs, const float* inputs,
                   std::size_t nW_rows, std::size_t nW_cols, const float* next_W,
                   const float* next_d, std::size_t next_d_len, float eta, float* deltas, float* G,
                   float* DW, float* db) {
    try {
        lane::FullyConnectedLayer L(in, out);
        std::memcpy(L.outputs.data.data(), outputs, out * sizeof(float));
        std::memcpy(L.inputs.data.data(), inputs, in * sizeof(float));
        lane::DenseMatrix nW(nW_rows, nW_cols);
        std::memcpy(nW.data.data(), next_W, nW_rows * nW_cols * sizeof(float));
        L.backward(nW, vec(next_d, next_d_len), lane::LearningRate(eta));
        std::memcpy(deltas, L.deltas.data.data(), out * sizeof(float));
        std::memcpy(G, L.gradients.data.data(), in * out * sizeof(float));
        std::memcpy(DW, L.delta_weights.data.data(), in * out * sizeof(float));
        std::memcpy(db, L.delta_biases.data.data(), out * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// FullyConnectedLayer / SoftmaxOutputLayer forward on a standalone layer.
int lr_layer_forward(int softmax, std::size_t in, std::size_t out, const float* W, const float* b,
                     const float* x, float* netin, float* outputs) {
    try {
        auto run = [&](auto& L) {
            std::memcpy(L.weights.data.data(), W, in * out * sizeof(float));
            std::memcpy(L.biases.data.data(), b, out * sizeof(float));
            L.forward(vec(x, in));
            std::memcpy(netin, L.netin.data.data(), out * sizeof(float));
            std::memcpy(outputs, L.outputs.data.data(), out * sizeof(float));
        };
        if (softmax) {
            lane::SoftmaxOutputLayer L(in, out);
            run(L);
        } else {
            lane::FullyConnectedLayer L(in, out);
            run(L);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int lr_train(void* netp, const float* X, const float* T, std::size_t n, float eta, float max_error,
             std::size_t max_epochs, std::uint64_t seed, int parallel, unsigned workers,
             float* loss, float* acc, std::size_t* epochs_run) {
    try {
        auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
        lane::DataSet d = make_set(X, T, n, net.input_width(), net.class_count());
        lane::TrainerConfig cfg;
        cfg.eta = lane::LearningRate(eta);
        cfg.max_error = max_error;
        cfg.max_epochs = max_epochs;
        cfg.seed = seed;
        lane::Device dev(kind_of(parallel), workers);
        auto stats = lane::train(net, d, cfg, dev);
        for (std::size_t e = 0; e < stats.size(); ++e) {
            loss[e] = stats[e].mean_loss;
            acc[e] = stats[e].accuracy;
        }
        *epochs_run = stats.size();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int lr_evaluate(void* netp, const float* X, const float* T, std::size_t n, float* loss,
                float* acc) {
    try {
        auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
        lane::DataSet d = make_set(X, T, n, net.input_width(), net.class_count());
        lane::EpochStats es = lane::evaluate(net, d);
        *loss = es.mean_loss;
        *acc = es.accuracy;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

float lr_cross_entropy(const float* p, const float* t, std::size_t n) {
    return lane::cross_entropy(vec(p, n), vec(t, n));
}

// The reference measure() loop (bench.cpp:55-73): per iteration one sample,
// net.forward + plan.run on one device.  Sample k = order[it] (order holds
// warmup + timed entries; null => it % n).  Returns the wall seconds of the timed iterations; the
// per-phase means (copy_in, kernel, copy_out summed over layers, forward) are
// written to phase_ms[4] when non-null.
double lr_sgd_bench(void* netp, const float* X, const float* T, std::size_t n,
                    const std::uint32_t* order, std::size_t warmup, std::size_t timed, float eta,
                    int parallel, unsigned workers, double* phase_ms) {
    try {
        auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
        const std::size_t F = net.input_width(), C = net.class_count();
        std::vector<lane::DenseVector> xs, ts;
        xs.reserve(n);
        ts.reserve(n);
        for (std::size_t k = 0; k < n; ++k) {
            xs.push_back(vec(X + k * F, F));
            ts.push_back(vec(T + k * C, C));
        }
        lane::Device dev(kind_of(parallel), workers);
        lane::BackwardPlan plan(net, lane::LearningRate(eta), dev);
        double ci = 0, kk = 0, co = 0, fw = 0;
        using clk = std::chrono::steady_clock;
        clk::time_point t0;
        for (std::size_t it = 0; it < warmup + timed; ++it) {
            if (it == warmup) t0 = clk::now();
            const std::size_t k = order ? order[it] : it % n;
            auto f0 = clk::now();
            net.forward(xs[k]);
            auto f1 = clk::now();
            auto pt = plan.run(ts[k]);
            if (it >= warmup) {
                fw += std::chrono::duration<double, std::milli>(f1 - f0).count();
                for (auto& p : pt) {
                    ci += p.copy_in_ms;
                    kk += p.kernel_ms;
                    co += p.copy_out_ms;
                }
            }
        }
        const double secs = std::chrono::duration<double>(clk::now() - t0).count();
        if (phase_ms && timed) {
            phase_ms[0] = ci / timed;
            phase_ms[1] = kk / timed;
            phase_ms[2] = co / timed;
            phase_ms[3] = fw / timed;
        }
        return secs;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

std::uint64_t lr_net_hash(void* netp) {
    auto& net = *static_cast<lane::FeedForwardNetwork*>(netp);
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (const auto& layer : net.hidden) {
        h = lane::fnv1a64(layer.weights.data.data(), layer.weights.data.size() * sizeof(float), h);
        h = lane::fnv1a64(layer.biases.data.data(), layer.biases.data.size() * sizeof(float), h);
    }
    h = lane::fnv1a64(net.output.weights.data.data(),
                      net.output.weights.data.size() * sizeof(float), h);
    h = lane::fnv1a64(net.output.biases.data.data(), net.output.biases.data.size() * sizeof(float),
                      h);
    return h;
}

void lr_rng_fill(std::uint64_t seed, std::size_t n, float lo, float hi, float* out) {
    lane::SeededRng rng(seed);
    lane::DenseVector v(n);
    lane::random_fill(v, rng, lo, hi);
    std::memcpy(out, v.data.data(), n * sizeof(float));
}

void lr_rng_u64(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    lane::SeededRng rng(seed);
    for (std::size_t k = 0; k < n; ++k) out[k] = rng.next_u64();
}

long lr_load_dataset(const char* path, std::size_t F, std::size_t C, float* X, float* T,
                     std::size_t cap) {
    try {
        lane::DataSet d = lane::load_dataset(path, F, C);
        if (d.size() > cap) return -1;
        for (std::size_t k = 0; k < d.size(); ++k) {
            std::memcpy(X + k * F, d.items[k].features.data.data(), F * sizeof(float));
            std::memcpy(T + k * C, d.items[k].label.data.data(), C * sizeof(float));
        }
        return static_cast<long>(d.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// split(d, frac, seed): writes train then test sets; returns the train count.
long lr_split(const float* X, const float* T, std::size_t n, std::size_t F, std::size_t C,
              double frac, std::uint64_t seed, float* Xo, float* To) {
    try {
        auto [tr, te] = lane::split(make_set(X, T, n, F, C), frac, seed);
        std::size_t k = 0;
        for (const auto* s : {&tr, &te})
            for (const auto& it : s->items) {
                std::memcpy(Xo + k * F, it.features.data.data(), F * sizeof(float));
                std::memcpy(To + k * C, it.label.data.data(), C * sizeof(float));
                ++k;
            }
        return static_cast<long>(tr.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

int lr_enlarge(const float* X, const float* T, std::size_t n, std::size_t F, std::size_t C,
               std::size_t factor, float noise, std::uint64_t seed, float* Xo, float* To) {
    try {
        lane::SeededRng rng(seed);
        lane::DataSet e = lane::enlarge(make_set(X, T, n, F, C), factor, noise, rng);
        for (std::size_t k = 0; k < e.size(); ++k) {
            std::memcpy(Xo + k * F, e.items[k].features.data.data(), F * sizeof(float));
            std::memcpy(To + k * C, e.items[k].label.data.data(), C * sizeof(float));
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"

// lane::run_benchmark + emit_report (bench.cpp:147-209): the reference's own
// lane-bench report (CSV) and final weights hash, for the B200 lane-bench
// parity test and bench.py's paper-table mode.  device: 0 serial, 1 parallel.
extern "C" long lr_run_benchmark(const char* dataset, std::size_t features, std::size_t classes,
                                 std::size_t fc_neurons, float eta, std::size_t warmup, std::size_t iters,
                                 std::size_t enlarge, int device, unsigned workers, std::uint64_t seed,
                                 char* csv, std::size_t csv_len, std::uint64_t* hash) {
    try {
        lane::BenchConfig cfg;
        cfg.dataset_path = dataset;
        cfg.features = features;
        cfg.classes = classes;
        cfg.fc_neurons = fc_neurons;
        cfg.eta = eta;
        cfg.warmup_iters = warmup;
        cfg.timed_iters = iters;
        cfg.enlarge_factor = enlarge;
        cfg.device = device ? lane::Device::Kind::ParallelHost : lane::Device::Kind::SerialHost;
        cfg.workers = workers;
        cfg.seed = seed;
        const lane::BenchReport rep = lane::run_benchmark(cfg);
        const std::string text = lane::emit_report(rep, lane::BenchConfig::Format::Csv);
        if (hash) *hash = rep.final_weights_hash;
        if (text.size() + 1 > csv_len) return -1;
        std::memcpy(csv, text.c_str(), text.size() + 1);
        return static_cast<long>(text.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}
