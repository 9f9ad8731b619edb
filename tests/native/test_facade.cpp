// The C++ facade (include/lane_b200/lane.hpp) driven like the reference's own
// doctest suites drive lane:: (proj/tests/test_layers.cpp, test_training.cpp).
// Built and run by tests/test_gpu_facade.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lane_b200/lane.hpp"

using namespace lane_b200;

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)      \
    do {                              \
        bool thrown = false;          \
        try {                         \
            expr;                     \
        } catch (const T&) {          \
            thrown = true;            \
        }                             \
        CHECK(thrown);                \
    } while (0)

static bool approx(float a, float b, float rel = 1e-6f) { return std::fabs(a - b) <= rel * std::fabs(b); }

int main(int argc, char** argv) {
    Device dev(0, Numerics::Strict);
    {
        // test_layers.cpp:125-142 softmax backward hand example
        FeedForwardNetwork net(dev, 3, {1}, 2);
        auto& out = net.output();
        out.write(LANE_BUF_OUTPUTS, {0.7f, 0.3f});
        out.write(LANE_BUF_INPUTS, {2.0f});
        out.backward({1.0f, 0.0f}, LearningRate(0.1f));
        auto d = out.deltas(), g = out.gradients(), dw = out.delta_weights(), db = out.delta_biases();
        CHECK(approx(d[0], -0.3f) && approx(d[1], 0.3f));
        CHECK(approx(g[0], -0.6f) && approx(g[1], 0.6f));
        CHECK(approx(dw[0], 0.06f) && approx(dw[1], -0.06f));
        CHECK(approx(db[0], 0.03f) && approx(db[1], -0.03f));
        CHECK_THROWS_AS(out.backward({1.0f}, LearningRate(0.1f)), ShapeError);
    }
    {
        // test_layers.cpp:209-222 fc backward hand example: delta = 0.45
        FeedForwardNetwork net(dev, 1, {1}, 2);
        auto& h = net.hidden[0];
        h.write(LANE_BUF_OUTPUTS, {0.5f});
        h.write(LANE_BUF_INPUTS, {1.0f});
        h.backward({3.0f}, 1, 1, {0.2f}, LearningRate(0.1f));
        CHECK(approx(h.deltas()[0], 0.45f));
        CHECK_THROWS_AS(h.backward({0.0f, 0.0f}, 2, 1, {0.2f}, LearningRate(0.1f)), ShapeError);
    }
    {
        // test_layers.cpp:240-258 apply_updates
        FeedForwardNetwork net(dev, 1, {1}, 2);
        auto& h = net.hidden[0];
        h.write(LANE_BUF_W, {1.0f});
        h.write(LANE_BUF_DW, {-0.06f});
        h.write(LANE_BUF_DELTA_BIASES, {0.5f});
        h.apply_updates();
        CHECK(h.weights()[0] == 0.94f && h.biases()[0] == 0.5f);
        h.apply_updates();
        CHECK(approx(h.weights()[0], 0.88f, 1e-6f));
    }
    {
        // test_layers.cpp:323-326 / network.cpp:28-40 config errors
        CHECK_THROWS_AS(LearningRate(0.0f), ConfigError);
        CHECK_THROWS_AS(FeedForwardNetwork(dev, 0, {}, 2), ConfigError);
        CHECK_THROWS_AS(FeedForwardNetwork(dev, 2, {0}, 2), ConfigError);
        CHECK_THROWS_AS(FeedForwardNetwork(dev, 2, {}, 1), ConfigError);
    }
    {
        // test_training.cpp:204-221 XOR regression oracle: 77 epochs, accuracy 1
        DataSet d;
        d.feature_width = 2;
        d.class_count = 2;
        d.features = {0, 0, 0, 1, 1, 0, 1, 1};
        d.labels = {1, 0, 0, 1, 0, 1, 1, 0};
        auto net = build_network(dev, 2, {4}, 2, 111);
        TrainerConfig cfg;
        cfg.eta = LearningRate(0.5f);
        cfg.max_epochs = 5000;
        cfg.max_error = 0.05f;
        cfg.seed = 111;
        auto stats = train(*net, d, cfg);
        CHECK(stats.size() == 77);
        CHECK(evaluate(*net, d).accuracy == 1.0f);
        // one BackwardPlan step lowers the loss (test_training.cpp:262-279)
        auto net2 = build_network(dev, 4, {5}, 3, 303);
        const std::vector<float> x = {0.1f, 0.7f, 0.3f, 0.9f}, t = {0.0f, 1.0f, 0.0f};
        const float before = -std::log(net2->forward(x)[1]);
        BackwardPlan(*net2, LearningRate(1e-3f)).run(t);
        const float after = -std::log(net2->forward(x)[1]);
        CHECK(after < before);
        DataSet empty;
        empty.feature_width = 2;
        empty.class_count = 2;
        CHECK_THROWS_AS(train(*net, empty, cfg), TrainingError);
    }
    if (argc > 1) {
        // dataset.hpp over the library loader: Iris, split(0.9, 42) -> 135/15
        // (acceptance.cpp:443-469), enlarge, save/load round trip, errors
        DataSet iris = load_dataset(argv[1], 4, 3);
        CHECK(iris.size() == 150);
        auto tt = split(iris, 0.9, 42);
        CHECK(tt.first.size() == 135 && tt.second.size() == 15);
        SeededRng rng(7);
        DataSet big = enlarge(tt.first, 3, 0.02f, rng);
        CHECK(big.size() == 405 && rng.state != 7);
        bool in_range = true;
        for (float v : big.features) in_range = in_range && v >= 0.0f && v <= 1.0f;
        CHECK(in_range);
        CHECK_THROWS_AS(split(iris, 1.0, 1), ConfigError);
        CHECK_THROWS_AS(enlarge(iris, 0, 0.1f, rng), ConfigError);
        CHECK_THROWS_AS(load_dataset("/nonexistent/iris.csv", 4, 3), IoError);
        CHECK_THROWS_AS(load_dataset(argv[1], 4, 2), ParseError);
        const std::string tmp = std::string(argc > 2 ? argv[2] : "/tmp") + "/facade_iris.csv";
        save_dataset(tt.second, tmp);
        DataSet back = load_dataset(tmp, 4, 3);
        CHECK(back.features == tt.second.features && back.labels == tt.second.labels);
        // mini-batch trainer over the loaded rows: the loss falls
        auto net = build_network(dev, 4, {16}, 3, 42, 16);
        auto losses = train_minibatch(*net, big, 16, LearningRate(0.1f), 0.9f, 20, 1);
        CHECK(losses.size() == 20 && losses.back() < 0.5f * losses.front());
        CHECK(evaluate(*net, tt.second).accuracy >= 0.8f);
    }
    if (failures == 0) std::printf("ALL PASSED\n");
    return failures == 0 ? 0 : 1;
}
