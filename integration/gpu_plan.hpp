// integration/gpu_plan.hpp -- the binding a maintainer of the reference adds
// to run its backward pass on a B200 through liblane_b200 (include/lane_b200.h).
//
// It is written against the REFERENCE's own headers (proj/include/lane/*.hpp)
// and types -- lane::FeedForwardNetwork, DenseVector, DataSet, PhaseTiming,
// LearningRate, the lane::Error hierarchy -- and is compiled and run against
// the reference library by tests/native/test_gpu_plan.cpp (oracle/Makefile,
// GPU test tests/test_gpu_plan.py).  Header-only; link liblane_b200.so.
//
// lane::GpuPlan has BackwardPlan's surface (proj/include/lane/network.hpp:58-75)
// in two residencies:
//
//   Residency::Mirror (default) -- a drop-in at the reference's own call sites,
//     e.g. measure() (proj/src/bench.cpp:62-72) and train's loop
//     (proj/src/network.cpp:164-170):
//         net.forward(s.features);   // host forward, unchanged
//         plan.run(s.label);         // backward + apply_updates on the GPU
//         ... hash_network(net) ...  // sees the update
//     The host network stays the source of truth, as with the reference's
//     TaskSchedule copy phases (src/task_runtime.cpp:240-303): run() copies
//     in the weights, biases and the forward cache (inputs / netin / outputs)
//     of every layer, runs BackwardPlan::run on the device, and copies every
//     LayerState buffer the reference's run() writes (weights, biases,
//     gradients, delta_weights, deltas, delta_biases) back.
//
//   Residency::Device -- the state lives in HBM; the forward runs on the
//     device too (plan.forward(x) instead of net.forward(x)), nothing crosses
//     PCIe per sample, and download() brings every LayerState buffer back
//     when the host needs it:
//         plan.forward(s.features);
//         plan.run(s.label);
//         ...
//         plan.download();  hash_network(net);
//
// train()/evaluate() run the library's fused epoch driver on the device
// (lane_b200_train / lane_b200_evaluate) and leave the host network current.
// With numerics STRICT (the default here) every result is bit-identical to
// the reference; FAST runs the fused kernels within DESIGN.md section 2's
// tolerance.
#pragma once

#include <chrono>
#include <cstddef>
#include <vector>

#include "lane/dataset.hpp"
#include "lane/error.hpp"
#include "lane/network.hpp"
#include "lane/task_runtime.hpp"
#include "lane_b200.h"

namespace lane {

class GpuPlan {
public:
    enum class Residency { Mirror, Device };

    GpuPlan(FeedForwardNetwork& net, LearningRate eta, int gpu = 0, Residency residency = Residency::Mirror,
            int numerics = LANE_NUMERICS_STRICT)
        : net_(net), eta_(eta), residency_(residency) {
        ok(lane_b200_ctx_create(gpu, &ctx_));
        ok(lane_b200_ctx_set_numerics(ctx_, numerics));
        std::vector<std::size_t> hidden;
        for (auto& l : net.hidden) hidden.push_back(l.cols_out());
        ok(lane_b200_net_create(ctx_, net.input_width(), hidden.data(), hidden.size(), net.class_count(), 1,
                                &gpu_));
        upload();
    }
    GpuPlan(const GpuPlan&) = delete;
    GpuPlan& operator=(const GpuPlan&) = delete;
    ~GpuPlan() {
        lane_b200_net_destroy(gpu_);
        lane_b200_ctx_destroy(ctx_);
    }

    Residency residency() const { return residency_; }

    // FeedForwardNetwork::forward on the device (Residency::Device); returns
    // the probabilities.  The host network is not touched.
    const DenseVector& forward(const DenseVector& input) {
        if (input.len() != net_.input_width()) throw ShapeError("forward: input length != input width");
        probs_.data.resize(net_.class_count());
        ok(lane_b200_forward(gpu_, input.data.data(), probs_.data.data()));
        return probs_;
    }

    // BackwardPlan::run (network.cpp:122-138): output layer, hidden layers in
    // reverse, then apply_updates on every layer.  One PhaseTiming per
    // schedule, output layer first (device-timed with CUDA events); in Mirror
    // residency the host<->device copies are the first schedule's copy_in /
    // copy_out, like the reference's per-execute copy phases.
    std::vector<PhaseTiming> run(const DenseVector& target) {
        if (target.len() != net_.class_count()) throw ShapeError("backward: target length != class count");
        using clock = std::chrono::steady_clock;
        double in_ms = 0.0, out_ms = 0.0;
        if (residency_ == Residency::Mirror) {
            const auto t0 = clock::now();
            for (std::size_t l = 0; l < layers(); ++l) {
                LayerState& L = layer(l);
                write(l, LANE_BUF_W, L.weights.data);
                write(l, LANE_BUF_B, L.biases.data);
                write(l, LANE_BUF_INPUTS, L.inputs.data);
                write(l, LANE_BUF_NETIN, L.netin.data);
                write(l, LANE_BUF_OUTPUTS, L.outputs.data);
            }
            in_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        }
        std::vector<double> ph(3 * layers());
        ok(lane_b200_backward_plan_run_timed(gpu_, target.data.data(), eta_.eta, ph.data(), ph.size()));
        if (residency_ == Residency::Mirror) {
            const auto t0 = clock::now();
            for (std::size_t l = 0; l < layers(); ++l) {
                LayerState& L = layer(l);
                read(l, LANE_BUF_W, L.weights.data);
                read(l, LANE_BUF_B, L.biases.data);
                read(l, LANE_BUF_G, L.gradients.data);
                read(l, LANE_BUF_DW, L.delta_weights.data);
                read(l, LANE_BUF_DELTAS, L.deltas.data);
                read(l, LANE_BUF_DELTA_BIASES, L.delta_biases.data);
            }
            out_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        }
        std::vector<PhaseTiming> out(layers());
        for (std::size_t k = 0; k < layers(); ++k) {
            out[k].copy_in_ms = ph[3 * k] + (k == 0 ? in_ms : 0.0);
            out[k].kernel_ms = ph[3 * k + 1];
            out[k].copy_out_ms = ph[3 * k + 2] + (k == 0 ? out_ms : 0.0);
            out[k].task_kernel_ms = {out[k].kernel_ms};
        }
        return out;
    }

    // lane::train (network.cpp:140-182) on the device: the reference's shuffle
    // stream, EpochStats, early stop.  The host network is current afterwards.
    std::vector<EpochStats> train(const DataSet& d, const TrainerConfig& cfg) {
        if (d.items.empty()) throw TrainingError("train: empty training set");
        if (d.feature_width != net_.input_width())
            throw ShapeError("train: dataset feature width != network input width");
        if (d.class_count != net_.class_count())
            throw ShapeError("train: dataset class count != network class count");
        if (residency_ == Residency::Mirror) upload();
        std::vector<float> X, T;
        flatten(d, X, T);
        std::vector<float> loss(cfg.max_epochs), acc(cfg.max_epochs);
        std::size_t ran = 0;
        ok(lane_b200_train(gpu_, X.data(), T.data(), d.size(), cfg.eta.eta, cfg.max_error, cfg.max_epochs, cfg.seed,
                           loss.data(), acc.data(), &ran));
        download();
        std::vector<EpochStats> out;
        for (std::size_t e = 0; e < ran; ++e) out.push_back({e + 1, loss[e], acc[e]});
        return out;
    }

    // lane::evaluate (network.cpp:184-204) on the device.
    EpochStats evaluate(const DataSet& d) {
        if (d.items.empty()) throw TrainingError("evaluate: empty test set");
        if (d.feature_width != net_.input_width() || d.class_count != net_.class_count())
            throw ShapeError("evaluate: dataset shape does not match network");
        if (residency_ == Residency::Mirror) upload();
        std::vector<float> X, T;
        flatten(d, X, T);
        EpochStats es;
        ok(lane_b200_evaluate(gpu_, X.data(), T.data(), d.size(), &es.mean_loss, &es.accuracy));
        return es;
    }

    // Every LayerState buffer, device -> host network.
    void download() {
        for (std::size_t l = 0; l < layers(); ++l) {
            LayerState& L = layer(l);
            read(l, LANE_BUF_W, L.weights.data);
            read(l, LANE_BUF_B, L.biases.data);
            read(l, LANE_BUF_G, L.gradients.data);
            read(l, LANE_BUF_DW, L.delta_weights.data);
            read(l, LANE_BUF_INPUTS, L.inputs.data);
            read(l, LANE_BUF_NETIN, L.netin.data);
            read(l, LANE_BUF_OUTPUTS, L.outputs.data);
            read(l, LANE_BUF_DELTAS, L.deltas.data);
            read(l, LANE_BUF_DELTA_BIASES, L.delta_biases.data);
        }
    }

    // Every LayerState buffer, host network -> device.
    void upload() {
        for (std::size_t l = 0; l < layers(); ++l) {
            LayerState& L = layer(l);
            write(l, LANE_BUF_W, L.weights.data);
            write(l, LANE_BUF_B, L.biases.data);
            write(l, LANE_BUF_G, L.gradients.data);
            write(l, LANE_BUF_DW, L.delta_weights.data);
            write(l, LANE_BUF_INPUTS, L.inputs.data);
            write(l, LANE_BUF_NETIN, L.netin.data);
            write(l, LANE_BUF_OUTPUTS, L.outputs.data);
            write(l, LANE_BUF_DELTAS, L.deltas.data);
            write(l, LANE_BUF_DELTA_BIASES, L.delta_biases.data);
        }
    }

private:
    // status codes 1..6 mirror lane::ShapeError .. ParseError (error.hpp:12-38)
    static void ok(int rc) {
        if (rc == LANE_OK) return;
        const char* m = lane_b200_last_error();
        switch (rc) {
            case LANE_ERR_SHAPE: throw ShapeError(m);
            case LANE_ERR_CONFIG: throw ConfigError(m);
            case LANE_ERR_SCHEDULE: throw ScheduleError(m);
            case LANE_ERR_TRAINING: throw TrainingError(m);
            case LANE_ERR_IO: throw IoError(m);
            case LANE_ERR_PARSE: throw ParseError(m);
            default: throw Error(m);
        }
    }
    std::size_t layers() const { return net_.hidden.size() + 1; }
    LayerState& layer(std::size_t l) {
        return l < net_.hidden.size() ? static_cast<LayerState&>(net_.hidden[l])
                                      : static_cast<LayerState&>(net_.output);
    }
    void write(std::size_t l, int buf, const std::vector<float>& v) {
        if (!v.empty()) ok(lane_b200_buf_write(gpu_, l, buf, v.data(), v.size()));
    }
    void read(std::size_t l, int buf, std::vector<float>& v) {
        if (!v.empty()) ok(lane_b200_buf_read(gpu_, l, buf, v.data(), v.size()));
    }
    static void flatten(const DataSet& d, std::vector<float>& X, std::vector<float>& T) {
        X.reserve(d.size() * d.feature_width);
        T.reserve(d.size() * d.class_count);
        for (const Sample& s : d.items) {
            X.insert(X.end(), s.features.data.begin(), s.features.data.end());
            T.insert(T.end(), s.label.data.begin(), s.label.data.end());
        }
    }

    FeedForwardNetwork& net_;
    LearningRate eta_;
    Residency residency_;
    lane_b200_ctx* ctx_ = nullptr;
    lane_b200_net* gpu_ = nullptr;
    DenseVector probs_;
};

}  // namespace lane
