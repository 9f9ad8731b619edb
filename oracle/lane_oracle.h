/*
 * lane_oracle.h -- CPU restatement of the reference's FC-backprop hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, smoke()
 * and bench.py's cpu_baseline leg compare the CUDA path against; the product
 * (paper_2001_04206_b200, liblane_b200.so) never links, loads or calls it.
 *
 * Every function restates one reference routine (file:line into
 * /root/reference/proj) in plain C with the reference's exact evaluation
 * order: fp32, ascending sequential sums, separately rounded multiply and add
 * (build with -ffp-contract=off: the reference objects contain no FMA), and
 * glibc libm for tanhf/expf/logf.  Pinned against the reference itself
 * (oracle/_ref/liblane_ref.so, built from the reference sources by
 * oracle/Makefile) and against the reference tests' known-answer vectors
 * -- see tests/test_oracle.py and tests/golden/make_golden.py.
 *
 * Extension (not in the reference): mini-batch
 * averaging and momentum, defined so that B=1, mu=0 reduces bit-for-bit to
 * the reference step (lo_minibatch_step).
 */
#ifndef LANE_ORACLE_H
#define LANE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64, proj/include/lane/tensor.hpp:13-44, proj/src/tensor.cpp:7-23 */
typedef struct {
    uint64_t seed;
    uint64_t state;
} lo_rng;

void lo_rng_init(lo_rng* r, uint64_t seed);
uint64_t lo_rng_next_u64(lo_rng* r);
float lo_rng_next_float(lo_rng* r);
float lo_rng_uniform(lo_rng* r, float lo, float hi);
size_t lo_rng_below(lo_rng* r, size_t n);
void lo_rng_split(lo_rng* r, lo_rng* child);
/* random_fill, proj/src/tensor.cpp:49-65 (row-major, one draw per element) */
void lo_random_fill(float* v, size_t n, lo_rng* r, float lo, float hi);

/* LayerState, proj/include/lane/layers.hpp:68-92, proj/src/layers.cpp:7-16.
 * W, G, DW are in x out row-major ([i*out + o]). */
typedef struct {
    size_t in, out;
    float* W;  /* weights       */
    float* G;  /* gradients     */
    float* DW; /* delta_weights */
    float* b;  /* biases        */
    float* x;  /* inputs        */
    float* z;  /* netin         */
    float* a;  /* outputs       */
    float* d;  /* deltas        */
    float* db; /* delta_biases  */
    /* extension: momentum velocity lives in DW */
} lo_layer;

int lo_layer_init(lo_layer* L, size_t in, size_t out);
void lo_layer_free(lo_layer* L);
void lo_layer_copy(lo_layer* dst, const lo_layer* src); /* same shape */

/* LayerState::compute_netin + FullyConnectedLayer::forward, layers.cpp:27-49 */
void lo_fc_forward(lo_layer* L, const float* x);
/* SoftmaxOutputLayer::forward, layers.cpp:71-87 */
void lo_softmax_forward(lo_layer* L, const float* x);
/* detail::softmax_backward_tuple over (o, i), layers.hpp:28-41, layers.cpp:89-102 */
void lo_softmax_backward(lo_layer* L, const float* target, float eta);
/* detail::fc_backward_tuple over (o, i), layers.hpp:43-61, layers.cpp:51-69.
 * next_W is out x next_out row-major (the next layer's weights). */
void lo_fc_backward(lo_layer* L, const float* next_W, size_t next_out,
                    const float* next_d, float eta);
/* LayerState::apply_updates, layers.cpp:18-25 */
void lo_apply_updates(lo_layer* L);

/* cross_entropy, network.cpp:68-79; argmax, network.cpp:13-21 */
float lo_cross_entropy(const float* p, const float* t, size_t n);
size_t lo_argmax(const float* v, size_t n);

/* FeedForwardNetwork, network.hpp:14-30; hidden[0..nh-1], then output */
typedef struct {
    size_t input_width;
    size_t n_hidden;
    lo_layer* layers; /* n_hidden + 1 entries; layers[n_hidden] = softmax output */
} lo_net;

/* build_network, network.cpp:55-66 (seeded from a fresh SeededRng(seed)) */
int lo_net_build(lo_net* net, size_t input_width, const size_t* hidden, size_t n_hidden,
                 size_t classes, uint64_t seed);
/* build_network with a caller-owned rng (so several nets can share one stream) */
int lo_net_build_rng(lo_net* net, size_t input_width, const size_t* hidden, size_t n_hidden,
                     size_t classes, lo_rng* rng);
void lo_net_free(lo_net* net);
void lo_net_copy(lo_net* dst, const lo_net* src); /* same topology */
/* FeedForwardNetwork::forward, network.cpp:47-53; returns output probabilities */
const float* lo_net_forward(lo_net* net, const float* x);
/* BackwardPlan::run, network.cpp:122-138: output backward, hidden backward in
 * reverse, then apply_updates on every hidden layer and the output. */
void lo_backward_plan_run(lo_net* net, const float* target, float eta);
/* Backward without the updates (acceptance.cpp:103-111 backward_no_update) */
void lo_backward_no_update(lo_net* net, const float* target, float eta);

typedef struct {
    size_t epoch;
    float mean_loss;
    float accuracy;
} lo_epoch_stats;

/* train, network.cpp:140-182.  X is n x input_width, T is n x classes.
 * Writes up to max_epochs stats; returns the number of epochs run. */
size_t lo_train(lo_net* net, const float* X, const float* T, size_t n, float eta,
                float max_error, size_t max_epochs, uint64_t seed, lo_epoch_stats* stats);
/* evaluate, network.cpp:184-204 */
lo_epoch_stats lo_evaluate(lo_net* net, const float* X, const float* T, size_t n);

/* Per-sample SGD over a sample stream (the bench measure() loop,
 * bench.cpp:62-70): sample s uses row order[s] (order has n_steps entries) or
 * s mod n when order is NULL; forward + BackwardPlan::run per sample.  Returns
 * the summed cross entropy (double). */
double lo_sgd_run(lo_net* net, const float* X, const float* T, size_t n, const uint32_t* order,
                  size_t n_steps, float eta);

/* Extension: one mini-batch step.  Per layer
 *   G   = (1/B) * sum_b delta_b (x) x_b        (b ascending, fp32)
 *   DW  = mu * DW + (-eta) * G                  (DW doubles as the velocity)
 *   W  += DW ; likewise for biases with db.
 * Every delta uses the pre-update weights.  B=1, mu=0 == lo_backward_plan_run.
 * Returns the summed cross entropy of the batch. */
double lo_minibatch_step(lo_net* net, const float* X, const float* T, size_t B, float eta,
                         float mu);

/* Dataset helpers, proj/src/dataset.cpp and proj/tests/test_support.hpp */
/* testsupport::synthetic_dataset, test_support.hpp:14-27 */
void lo_synthetic_dataset(size_t features, size_t classes, size_t count, uint64_t seed, float* X,
                          float* T);
/* load_dataset, dataset.cpp:31-83 (strtof == from_chars rounding).  Returns the
 * number of samples written (<= cap) or -1 on error. */
long lo_load_dataset(const char* path, size_t features, size_t classes, float* X, float* T,
                     size_t cap);
/* split, dataset.cpp:103-124: writes the permutation; returns train count */
size_t lo_split_order(size_t n, double train_fraction, uint64_t seed, uint32_t* order);
/* enlarge, dataset.cpp:126-148 */
void lo_enlarge(const float* X, const float* T, size_t n, size_t features, size_t classes,
                size_t factor, float noise, lo_rng* rng, float* Xo, float* To);

/* bench.cpp:138-140 fnv1a64 */
uint64_t lo_fnv1a64(const void* data, size_t len, uint64_t seed);
uint64_t lo_net_hash(const lo_net* net);

/* Handle helpers for FFI callers (tests, bench cpu_baseline). */
lo_net* lo_net_new(size_t in, const size_t* hidden, size_t nh, size_t classes, uint64_t seed);
lo_net* lo_net_clone(const lo_net* src);
void lo_net_delete(lo_net* net);
float* lo_net_buf(lo_net* net, size_t layer, int buf, size_t* count);
lo_layer* lo_layer_new(size_t in, size_t out);
void lo_layer_delete(lo_layer* L);

#ifdef __cplusplus
}
#endif

#endif
