// The reference-side binding (integration/gpu_plan.hpp) compiled against the
// REFERENCE's headers and linked with the reference library built from its
// own sources (oracle/Makefile -> oracle/_ref/test_gpu_plan; test
// infrastructure).  It runs the reference's measure() loop
// (proj/src/bench.cpp:62-72) and train() (proj/src/network.cpp:140-182)
// twice -- once with lane::BackwardPlan on a SerialHost Device, once with
// lane::GpuPlan -- and requires STRICT parity: the FNV-1a weights hash of
// hash_network (bench.cpp:32-41) and every LayerState buffer bit-identical.
// Run by tests/test_gpu_plan.py on the GPU box; prints "gpu_plan ok" and
// exits 0 on success.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gpu_plan.hpp"
#include "lane/bench.hpp"
#include "lane/network.hpp"

using namespace lane;

static int failures = 0;
#define CHECK(c, what)                                                                  \
    do {                                                                                \
        if (!(c)) {                                                                     \
            std::printf("FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #c, (what).c_str()); \
            ++failures;                                                                 \
        }                                                                               \
    } while (0)

// bench.cpp:32-41 (file-local there)
static std::uint64_t hash_network(const FeedForwardNetwork& net) {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (const auto& layer : net.hidden) {
        h = fnv1a64(layer.weights.data.data(), layer.weights.data.size() * sizeof(float), h);
        h = fnv1a64(layer.biases.data.data(), layer.biases.data.size() * sizeof(float), h);
    }
    h = fnv1a64(net.output.weights.data.data(), net.output.weights.data.size() * sizeof(float), h);
    h = fnv1a64(net.output.biases.data.data(), net.output.biases.data.size() * sizeof(float), h);
    return h;
}

// testsupport::synthetic_dataset (proj/tests/test_support.hpp:14-27)
static DataSet synthetic(std::size_t F, std::size_t C, std::size_t n, std::uint64_t seed) {
    SeededRng rng(seed);
    DataSet d;
    d.feature_width = F;
    d.class_count = C;
    for (std::size_t k = 0; k < n; ++k) {
        Sample s{DenseVector(F), DenseVector(C)};
        for (std::size_t i = 0; i < F; ++i) s.features[i] = rng.next_float();
        s.label[rng.below(C)] = 1.0f;
        d.items.push_back(std::move(s));
    }
    return d;
}

static bool same(const std::vector<float>& a, const std::vector<float>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

static void check_buffers(const FeedForwardNetwork& a, const FeedForwardNetwork& b, const std::string& what) {
    for (std::size_t l = 0; l <= a.hidden.size(); ++l) {
        const LayerState& x = l < a.hidden.size() ? static_cast<const LayerState&>(a.hidden[l]) : a.output;
        const LayerState& y = l < b.hidden.size() ? static_cast<const LayerState&>(b.hidden[l]) : b.output;
        const std::string w = what + " layer " + std::to_string(l);
        CHECK(same(x.weights.data, y.weights.data), w + " weights");
        CHECK(same(x.biases.data, y.biases.data), w + " biases");
        CHECK(same(x.gradients.data, y.gradients.data), w + " gradients");
        CHECK(same(x.delta_weights.data, y.delta_weights.data), w + " delta_weights");
        CHECK(same(x.deltas.data, y.deltas.data), w + " deltas");
        CHECK(same(x.delta_biases.data, y.delta_biases.data), w + " delta_biases");
    }
}

struct Shape {
    std::size_t F;
    std::vector<std::size_t> H;
    std::size_t C;
    float eta;
    std::size_t iters;
};

int main() {
    const Shape shapes[] = {
        {784, {128}, 10, 0.01f, 60},      // C2, the paper-style single hidden layer
        {4, {8}, 3, 0.1f, 200},           // C1
        {340, {1024}, 10, 1e-4f, 20},     // C4 width sweep point
        {20, {16, 12}, 5, 0.05f, 100},    // two hidden layers
    };
    for (const Shape& sh : shapes) {
        const std::string name = std::to_string(sh.F) + "-" + std::to_string(sh.H[0]) + "-" + std::to_string(sh.C);
        const DataSet ds = synthetic(sh.F, sh.C, 32, 9);

        // the reference: measure()'s loop with BackwardPlan on SerialHost
        SeededRng r0(42);
        FeedForwardNetwork ref = build_network(sh.F, sh.H, sh.C, r0);
        Device host(Device::Kind::SerialHost);
        BackwardPlan plan(ref, LearningRate(sh.eta), host);
        for (std::size_t it = 0; it < sh.iters; ++it) {
            const Sample& s = ds.items[it % ds.items.size()];
            ref.forward(s.features);
            plan.run(s.label);
        }
        const std::uint64_t want = hash_network(ref);

        // GpuPlan at the same call site (Mirror residency): host forward,
        // device backward + update, host network current after every run()
        SeededRng r1(42);
        FeedForwardNetwork mir = build_network(sh.F, sh.H, sh.C, r1);
        {
            GpuPlan gp(mir, LearningRate(sh.eta));
            for (std::size_t it = 0; it < sh.iters; ++it) {
                const Sample& s = ds.items[it % ds.items.size()];
                mir.forward(s.features);
                const std::vector<PhaseTiming> t = gp.run(s.label);
                CHECK(t.size() == sh.H.size() + 1, name + " PhaseTiming per schedule");
            }
        }
        CHECK(hash_network(mir) == want, name + " mirror hash");
        check_buffers(mir, ref, name + " mirror");

        // Device residency: forward on the device too, one download at the end
        SeededRng r2(42);
        FeedForwardNetwork dev = build_network(sh.F, sh.H, sh.C, r2);
        {
            GpuPlan gp(dev, LearningRate(sh.eta), 0, GpuPlan::Residency::Device);
            for (std::size_t it = 0; it < sh.iters; ++it) {
                const Sample& s = ds.items[it % ds.items.size()];
                const DenseVector& p = gp.forward(s.features);
                CHECK(p.len() == sh.C, name + " probabilities");
                gp.run(s.label);
            }
            gp.download();
        }
        CHECK(hash_network(dev) == want, name + " device hash");
        check_buffers(dev, ref, name + " device");

        // train() and evaluate(): the reference's epoch driver vs the device's
        TrainerConfig cfg{LearningRate(sh.eta), 0.0f, 3, 42};
        SeededRng r3(42), r4(42);
        FeedForwardNetwork tr = build_network(sh.F, sh.H, sh.C, r3);
        FeedForwardNetwork tg = build_network(sh.F, sh.H, sh.C, r4);
        const std::vector<EpochStats> es_ref = train(tr, ds, cfg, host);
        std::vector<EpochStats> es_gpu;
        EpochStats ev_gpu;
        {
            GpuPlan gp(tg, LearningRate(sh.eta));
            es_gpu = gp.train(ds, cfg);
            ev_gpu = gp.evaluate(ds);
        }
        CHECK(es_ref.size() == es_gpu.size(), name + " epochs run");
        for (std::size_t e = 0; e < es_ref.size() && e < es_gpu.size(); ++e) {
            CHECK(std::memcmp(&es_ref[e].mean_loss, &es_gpu[e].mean_loss, 4) == 0, name + " epoch loss");
            CHECK(std::memcmp(&es_ref[e].accuracy, &es_gpu[e].accuracy, 4) == 0, name + " epoch accuracy");
        }
        CHECK(hash_network(tg) == hash_network(tr), name + " train hash");
        const EpochStats ev_ref = evaluate(tr, ds);
        CHECK(std::memcmp(&ev_ref.mean_loss, &ev_gpu.mean_loss, 4) == 0, name + " evaluate loss");
        CHECK(std::memcmp(&ev_ref.accuracy, &ev_gpu.accuracy, 4) == 0, name + " evaluate accuracy");
        std::printf("%s: %zu measure() iterations, hash %016llx; %zu epochs\n", name.c_str(), sh.iters,
                    static_cast<unsigned long long>(want), es_ref.size());
    }

    // the reference's error classes cross the boundary
    {
        SeededRng r(1);
        FeedForwardNetwork net = build_network(6, {4}, 3, r);
        GpuPlan gp(net, LearningRate(0.1f));
        bool shape = false;
        try {
            gp.run(DenseVector(2));
        } catch (const ShapeError&) {
            shape = true;
        }
        CHECK(shape, std::string("ShapeError for a short target"));
        bool training = false;
        try {
            gp.train(DataSet{6, 3, {}}, TrainerConfig{});
        } catch (const TrainingError&) {
            training = true;
        }
        CHECK(training, std::string("TrainingError for an empty set"));
    }
    if (failures) {
        std::printf("%d failures\n", failures);
        return 1;
    }
    std::printf("gpu_plan ok\n");
    return 0;
}
