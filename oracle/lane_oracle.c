/*
 * lane_oracle.c -- CPU restatement of the reference FC-backprop hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lane_oracle.h).  Compiled by oracle/Makefile
 * with -O2 -ffp-contract=off so every a*b+c rounds twice, exactly like the
 * reference objects (baseline x86-64, no -march, no FMA).
 * Citations are path:line into /root/reference/proj.
 */
#include "lane_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng --- */

void lo_rng_init(lo_rng* r, uint64_t seed) {
    r->seed = seed;
    r->state = seed;
}

/* include/lane/tensor.hpp:19-25 */
uint64_t lo_rng_next_u64(lo_rng* r) {
    r->state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* include/lane/tensor.hpp:28-30: 24-bit resolution, exact in float */
float lo_rng_next_float(lo_rng* r) { return (float)(lo_rng_next_u64(r) >> 40) * 0x1p-24f; }

/* src/tensor.cpp:7-15: half-open [lo, hi) even when the scale rounds up */
float lo_rng_uniform(lo_rng* r, float lo, float hi) {
    float v = lo + lo_rng_next_float(r) * (hi - lo);
    return v < hi ? v : nextafterf(hi, lo);
}

/* src/tensor.cpp:17-23: Lemire multiply-shift, no rejection */
size_t lo_rng_below(lo_rng* r, size_t n) {
    return (size_t)(((unsigned __int128)lo_rng_next_u64(r) * (unsigned __int128)n) >> 64);
}

/* include/lane/tensor.hpp:39 */
void lo_rng_split(lo_rng* r, lo_rng* child) {
    lo_rng_init(child, lo_rng_next_u64(r) ^ 0x9E3779B97F4A7C15ULL);
}

/* src/tensor.cpp:49-56 */
void lo_random_fill(float* v, size_t n, lo_rng* r, float lo, float hi) {
    for (size_t k = 0; k < n; ++k) v[k] = lo_rng_uniform(r, lo, hi);
}

/* -------------------------------------------------------------- layer --- */

int lo_layer_init(lo_layer* L, size_t in, size_t out) {
    memset(L, 0, sizeof(*L));
    L->in = in;
    L->out = out;
    L->W = calloc(in * out, sizeof(float));
    L->G = calloc(in * out, sizeof(float));
    L->DW = calloc(in * out, sizeof(float));
    L->b = calloc(out, sizeof(float));
    L->x = calloc(in, sizeof(float));
    L->z = calloc(out, sizeof(float));
    L->a = calloc(out, sizeof(float));
    L->d = calloc(out, sizeof(float));
    L->db = calloc(out, sizeof(float));
    return (L->W && L->G && L->DW && L->b && L->x && L->z && L->a && L->d && L->db) ? 0 : -1;
}

void lo_layer_free(lo_layer* L) {
    free(L->W); free(L->G); free(L->DW); free(L->b); free(L->x);
    free(L->z); free(L->a); free(L->d); free(L->db);
    memset(L, 0, sizeof(*L));
}

void lo_layer_copy(lo_layer* dst, const lo_layer* s) {
    const size_t m = s->in * s->out * sizeof(float), v = s->out * sizeof(float);
    memcpy(dst->W, s->W, m); memcpy(dst->G, s->G, m); memcpy(dst->DW, s->DW, m);
    memcpy(dst->b, s->b, v); memcpy(dst->x, s->x, s->in * sizeof(float));
    memcpy(dst->z, s->z, v); memcpy(dst->a, s->a, v); memcpy(dst->d, s->d, v);
    memcpy(dst->db, s->db, v);
}

/* src/layers.cpp:27-41: netin[j] = (sum_{i asc} x_i*W[i][j]) + b_j; caches x */
static void compute_netin(lo_layer* L, const float* x) {
    if (L->x != x) memcpy(L->x, x, L->in * sizeof(float));
    for (size_t j = 0; j < L->out; ++j) {
        float sum = 0.0f;
        for (size_t i = 0; i < L->in; ++i) sum += L->x[i] * L->W[i * L->out + j];
        L->z[j] = sum + L->b[j];
    }
}

/* src/layers.cpp:43-49 */
void lo_fc_forward(lo_layer* L, const float* x) {
    compute_netin(L, x);
    for (size_t j = 0; j < L->out; ++j) L->a[j] = tanhf(L->z[j]);
}

/* src/layers.cpp:71-87: max-subtracted softmax, sequential sum */
void lo_softmax_forward(lo_layer* L, const float* x) {
    compute_netin(L, x);
    float mx = L->z[0];
    for (size_t j = 1; j < L->out; ++j) mx = L->z[j] > mx ? L->z[j] : mx; /* std::max */
    float sum = 0.0f;
    for (size_t j = 0; j < L->out; ++j) {
        L->a[j] = expf(L->z[j] - mx);
        sum += L->a[j];
    }
    for (size_t j = 0; j < L->out; ++j) L->a[j] /= sum;
}

/* include/lane/layers.hpp:28-41 over o-outer / i-inner (src/layers.cpp:97-101) */
void lo_softmax_backward(lo_layer* L, const float* t, float eta) {
    const size_t O = L->out;
    for (size_t o = 0; o < O; ++o) {
        const float delta = L->a[o] - t[o];
        for (size_t i = 0; i < L->in; ++i) {
            const float grad = delta * L->x[i];
            L->G[i * O + o] = grad;
            L->DW[i * O + o] = -eta * grad;
        }
        L->d[o] = delta;
        L->db[o] = -eta * delta;
    }
}

/* include/lane/layers.hpp:43-61.  The reference recomputes the k-sum for every
 * i (layers.hpp:49-52); it is the same deterministic sequence each time, so
 * computing it once per o is bit-identical. */
void lo_fc_backward(lo_layer* L, const float* nW, size_t nO, const float* nd, float eta) {
    const size_t O = L->out;
    for (size_t o = 0; o < O; ++o) {
        float weighted = 0.0f;
        for (size_t k = 0; k < nO; ++k) weighted += nd[k] * nW[o * nO + k];
        const float delta = (1.0f - L->a[o] * L->a[o]) * weighted;
        for (size_t i = 0; i < L->in; ++i) {
            const float grad = delta * L->x[i];
            L->G[i * O + o] = grad;
            L->DW[i * O + o] = -eta * grad;
        }
        L->d[o] = delta;
        L->db[o] = -eta * delta;
    }
}

/* src/layers.cpp:18-25 */
void lo_apply_updates(lo_layer* L) {
    const size_t n = L->in * L->out;
    for (size_t k = 0; k < n; ++k) L->W[k] += L->DW[k];
    for (size_t j = 0; j < L->out; ++j) L->b[j] += L->db[j];
}

/* ------------------------------------------------------------ network --- */

/* src/network.cpp:68-79 */
float lo_cross_entropy(const float* p, const float* t, size_t n) {
    float loss = 0.0f;
    for (size_t o = 0; o < n; ++o) {
        if (t[o] != 0.0f) {
            const float q = p[o] < 1e-12f ? 1e-12f : p[o]; /* std::max(p, 1e-12f) */
            loss -= t[o] * logf(q);
        }
    }
    return loss;
}

/* src/network.cpp:13-21: ties resolve to the lowest index */
size_t lo_argmax(const float* v, size_t n) {
    size_t best = 0;
    for (size_t i = 1; i < n; ++i)
        if (v[i] > v[best]) best = i;
    return best;
}

int lo_net_build_rng(lo_net* net, size_t in, const size_t* hidden, size_t nh, size_t classes,
                     lo_rng* rng) {
    if (in == 0 || classes < 2) return -1;
    for (size_t l = 0; l < nh; ++l)
        if (hidden[l] == 0) return -1;
    net->input_width = in;
    net->n_hidden = nh;
    net->layers = calloc(nh + 1, sizeof(lo_layer));
    size_t w = in;
    for (size_t l = 0; l < nh; ++l) {
        if (lo_layer_init(&net->layers[l], w, hidden[l])) return -1;
        w = hidden[l];
    }
    if (lo_layer_init(&net->layers[nh], w, classes)) return -1;
    /* src/network.cpp:58-64: hidden layers in order, then the output */
    for (size_t l = 0; l <= nh; ++l) {
        lo_layer* L = &net->layers[l];
        const float bound = 1.0f / sqrtf((float)L->in);
        lo_random_fill(L->W, L->in * L->out, rng, -bound, bound);
    }
    return 0;
}

int lo_net_build(lo_net* net, size_t in, const size_t* hidden, size_t nh, size_t classes,
                 uint64_t seed) {
    lo_rng rng;
    lo_rng_init(&rng, seed);
    return lo_net_build_rng(net, in, hidden, nh, classes, &rng);
}

void lo_net_free(lo_net* net) {
    if (!net->layers) return;
    for (size_t l = 0; l <= net->n_hidden; ++l) lo_layer_free(&net->layers[l]);
    free(net->layers);
    net->layers = NULL;
}

void lo_net_copy(lo_net* dst, const lo_net* src) {
    for (size_t l = 0; l <= src->n_hidden; ++l) lo_layer_copy(&dst->layers[l], &src->layers[l]);
}

/* src/network.cpp:47-53 */
const float* lo_net_forward(lo_net* net, const float* x) {
    const float* a = x;
    for (size_t l = 0; l < net->n_hidden; ++l) {
        lo_fc_forward(&net->layers[l], a);
        a = net->layers[l].a;
    }
    lo_softmax_forward(&net->layers[net->n_hidden], a);
    return net->layers[net->n_hidden].a;
}

void lo_backward_no_update(lo_net* net, const float* t, float eta) {
    const size_t nh = net->n_hidden;
    lo_softmax_backward(&net->layers[nh], t, eta);
    for (size_t l = nh; l-- > 0;) {
        const lo_layer* next = &net->layers[l + 1];
        lo_fc_backward(&net->layers[l], next->W, next->out, next->d, eta);
    }
}

/* src/network.cpp:122-138 */
void lo_backward_plan_run(lo_net* net, const float* t, float eta) {
    lo_backward_no_update(net, t, eta);
    for (size_t l = 0; l < net->n_hidden; ++l) lo_apply_updates(&net->layers[l]);
    lo_apply_updates(&net->layers[net->n_hidden]);
}

/* src/network.cpp:140-182 */
size_t lo_train(lo_net* net, const float* X, const float* T, size_t n, float eta,
                float max_error, size_t max_epochs, uint64_t seed, lo_epoch_stats* stats) {
    if (n == 0) return 0;
    const size_t I = net->input_width, C = net->layers[net->n_hidden].out;
    lo_rng rng;
    lo_rng_init(&rng, seed);
    size_t* order = malloc(n * sizeof(size_t));
    for (size_t k = 0; k < n; ++k) order[k] = k;
    size_t ran = 0;
    for (size_t epoch = 1; epoch <= max_epochs; ++epoch) {
        /* network.cpp:159-161: order is NOT reset, each epoch permutes the last */
        for (size_t i = n; i > 1; --i) {
            const size_t j = lo_rng_below(&rng, i);
            const size_t tmp = order[i - 1];
            order[i - 1] = order[j];
            order[j] = tmp;
        }
        double loss_sum = 0.0;
        size_t correct = 0;
        for (size_t k = 0; k < n; ++k) {
            const float* x = X + order[k] * I;
            const float* t = T + order[k] * C;
            const float* p = lo_net_forward(net, x);
            loss_sum += (double)lo_cross_entropy(p, t, C);
            correct += lo_argmax(p, C) == lo_argmax(t, C) ? 1 : 0;
            lo_backward_plan_run(net, t, eta);
        }
        lo_epoch_stats es;
        es.epoch = epoch;
        es.mean_loss = (float)(loss_sum / (double)n);
        es.accuracy = (float)correct / (float)n;
        stats[ran++] = es;
        if (es.mean_loss <= max_error) break;
    }
    free(order);
    return ran;
}

/* src/network.cpp:184-204 */
lo_epoch_stats lo_evaluate(lo_net* net, const float* X, const float* T, size_t n) {
    const size_t I = net->input_width, C = net->layers[net->n_hidden].out;
    double loss_sum = 0.0;
    size_t correct = 0;
    for (size_t k = 0; k < n; ++k) {
        const float* p = lo_net_forward(net, X + k * I);
        loss_sum += (double)lo_cross_entropy(p, T + k * C, C);
        correct += lo_argmax(p, C) == lo_argmax(T + k * C, C) ? 1 : 0;
    }
    lo_epoch_stats es;
    es.epoch = 0;
    es.mean_loss = (float)(loss_sum / (double)n);
    es.accuracy = (float)correct / (float)n;
    return es;
}

double lo_sgd_run(lo_net* net, const float* X, const float* T, size_t n, const uint32_t* order,
                  size_t n_steps, float eta) {
    const size_t I = net->input_width, C = net->layers[net->n_hidden].out;
    double loss = 0.0;
    for (size_t s = 0; s < n_steps; ++s) {
        const size_t k = order ? order[s] : s % n;
        const float* p = lo_net_forward(net, X + k * I);
        loss += (double)lo_cross_entropy(p, T + k * C, C);
        lo_backward_plan_run(net, T + k * C, eta);
    }
    return loss;
}

/* ------------------------------------------------- extension: batches --- */

double lo_minibatch_step(lo_net* net, const float* X, const float* T, size_t B, float eta,
                         float mu) {
    const size_t nh = net->n_hidden, I = net->input_width, C = net->layers[nh].out;
    /* accumulators: gradient sums per layer, bias sums per layer; the
     * velocities (DW, db) are saved first because the per-sample reference
     * backward overwrites delta_weights/delta_biases (layers.hpp:35, :39). */
    float** gsum = calloc(nh + 1, sizeof(float*));
    float** bsum = calloc(nh + 1, sizeof(float*));
    float** vW = calloc(nh + 1, sizeof(float*));
    float** vb = calloc(nh + 1, sizeof(float*));
    for (size_t l = 0; l <= nh; ++l) {
        const size_t m = net->layers[l].in * net->layers[l].out, o = net->layers[l].out;
        gsum[l] = calloc(m, sizeof(float));
        bsum[l] = calloc(o, sizeof(float));
        vW[l] = malloc(m * sizeof(float));
        vb[l] = malloc(o * sizeof(float));
        memcpy(vW[l], net->layers[l].DW, m * sizeof(float));
        memcpy(vb[l], net->layers[l].db, o * sizeof(float));
    }
    double loss = 0.0;
    for (size_t s = 0; s < B; ++s) {
        const float* p = lo_net_forward(net, X + s * I);
        loss += (double)lo_cross_entropy(p, T + s * C, C);
        lo_backward_no_update(net, T + s * C, eta);
        for (size_t l = 0; l <= nh; ++l) {
            const lo_layer* L = &net->layers[l];
            for (size_t i = 0; i < L->in; ++i)
                for (size_t o = 0; o < L->out; ++o)
                    gsum[l][i * L->out + o] += L->d[o] * L->x[i];
            for (size_t o = 0; o < L->out; ++o) bsum[l][o] += L->d[o];
        }
    }
    const float invB = 1.0f / (float)B;
    for (size_t l = 0; l <= nh; ++l) {
        lo_layer* L = &net->layers[l];
        const size_t n = L->in * L->out;
        for (size_t k = 0; k < n; ++k) {
            const float g = gsum[l][k] * invB;
            L->G[k] = g;
            L->DW[k] = mu == 0.0f ? -eta * g : mu * vW[l][k] + -eta * g;
            L->W[k] += L->DW[k];
        }
        for (size_t o = 0; o < L->out; ++o) {
            const float g = bsum[l][o] * invB;
            L->db[o] = mu == 0.0f ? -eta * g : mu * vb[l][o] + -eta * g;
            L->b[o] += L->db[o];
        }
        free(gsum[l]);
        free(bsum[l]);
        free(vW[l]);
        free(vb[l]);
    }
    free(gsum);
    free(bsum);
    free(vW);
    free(vb);
    return loss;
}

/* ----------------------------------------------------------- datasets --- */

/* tests/test_support.hpp:14-27 */
void lo_synthetic_dataset(size_t F, size_t C, size_t count, uint64_t seed, float* X, float* T) {
    lo_rng rng;
    lo_rng_init(&rng, seed);
    for (size_t n = 0; n < count; ++n) {
        lo_random_fill(X + n * F, F, &rng, 0.0f, 1.0f);
        memset(T + n * C, 0, C * sizeof(float));
        T[n * C + lo_rng_below(&rng, C)] = 1.0f;
    }
}

/* src/dataset.cpp:31-83.  strtof rounds the decimal directly to float like
 * std::from_chars<float>. */
long lo_load_dataset(const char* path, size_t F, size_t C, float* X, float* T, size_t cap) {
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    char line[8192];
    long count = 0;
    while (fgets(line, sizeof line, f)) {
        size_t len = strlen(line);
        while (len && (line[len - 1] == '\n' || line[len - 1] == '\r')) line[--len] = 0;
        if (!len) continue;
        if ((size_t)count >= cap) { fclose(f); return -1; }
        char* p = line;
        size_t ones = 0;
        for (size_t k = 0; k < F + C; ++k) {
            char* end;
            const float v = strtof(p, &end);
            if (end == p || (*end != ',' && *end != 0) || (*end == 0 && k + 1 < F + C)) {
                fclose(f);
                return -1;
            }
            if (k < F) {
                X[count * F + k] = v;
            } else {
                if (v != 0.0f && v != 1.0f) { fclose(f); return -1; }
                ones += v == 1.0f;
                T[count * C + (k - F)] = v;
            }
            p = *end ? end + 1 : end;
        }
        if (*p != 0 || ones != 1) { fclose(f); return -1; }
        ++count;
    }
    fclose(f);
    return count;
}

/* src/dataset.cpp:103-124 */
size_t lo_split_order(size_t n, double frac, uint64_t seed, uint32_t* order) {
    for (size_t k = 0; k < n; ++k) order[k] = (uint32_t)k;
    lo_rng rng;
    lo_rng_init(&rng, seed);
    for (size_t i = n; i > 1; --i) {
        const size_t j = lo_rng_below(&rng, i);
        const uint32_t tmp = order[i - 1];
        order[i - 1] = order[j];
        order[j] = tmp;
    }
    return (size_t)floor(frac * (double)n);
}

/* src/dataset.cpp:126-148 */
void lo_enlarge(const float* X, const float* T, size_t n, size_t F, size_t C, size_t factor,
                float noise, lo_rng* rng, float* Xo, float* To) {
    size_t out = 0;
    for (size_t s = 0; s < n; ++s) {
        for (size_t r = 0; r < factor; ++r, ++out) {
            for (size_t k = 0; k < F; ++k) {
                float x = X[s * F + k];
                if (noise > 0.0f) {
                    x = x + lo_rng_uniform(rng, -noise, noise);
                    x = x < 0.0f ? 0.0f : (x > 1.0f ? 1.0f : x); /* std::clamp */
                }
                Xo[out * F + k] = x;
            }
            memcpy(To + out * C, T + s * C, C * sizeof(float));
        }
    }
}

/* src/bench.cpp:138-146 */
uint64_t lo_fnv1a64(const void* data, size_t len, uint64_t h) {
    const unsigned char* b = data;
    for (size_t i = 0; i < len; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* src/bench.cpp:32-41: hidden (W, b) in order, then output (W, b) */
uint64_t lo_net_hash(const lo_net* net) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t l = 0; l <= net->n_hidden; ++l) {
        const lo_layer* L = &net->layers[l];
        h = lo_fnv1a64(L->W, L->in * L->out * sizeof(float), h);
        h = lo_fnv1a64(L->b, L->out * sizeof(float), h);
    }
    return h;
}

/* ------------------------------------------------ handle helpers (FFI) --- */

lo_net* lo_net_new(size_t in, const size_t* hidden, size_t nh, size_t classes, uint64_t seed) {
    lo_net* net = calloc(1, sizeof(lo_net));
    if (!net || lo_net_build(net, in, hidden, nh, classes, seed)) {
        if (net) lo_net_free(net);
        free(net);
        return NULL;
    }
    return net;
}

lo_net* lo_net_clone(const lo_net* src) {
    size_t* hidden = malloc((src->n_hidden + 1) * sizeof(size_t));
    for (size_t l = 0; l < src->n_hidden; ++l) hidden[l] = src->layers[l].out;
    lo_net* net = lo_net_new(src->input_width, hidden, src->n_hidden,
                             src->layers[src->n_hidden].out, 0);
    free(hidden);
    if (net) lo_net_copy(net, src);
    return net;
}

void lo_net_delete(lo_net* net) {
    if (!net) return;
    lo_net_free(net);
    free(net);
}

/* Buffer ids follow include/lane_b200.h (LANE_BUF_*): 0 W, 1 G, 2 DW, 3 b,
 * 4 inputs, 5 netin, 6 outputs, 7 deltas, 8 delta_biases. */
float* lo_net_buf(lo_net* net, size_t layer, int buf, size_t* count) {
    if (layer > net->n_hidden) return NULL;
    lo_layer* L = &net->layers[layer];
    const size_t m = L->in * L->out;
    switch (buf) {
        case 0: *count = m; return L->W;
        case 1: *count = m; return L->G;
        case 2: *count = m; return L->DW;
        case 3: *count = L->out; return L->b;
        case 4: *count = L->in; return L->x;
        case 5: *count = L->out; return L->z;
        case 6: *count = L->out; return L->a;
        case 7: *count = L->out; return L->d;
        case 8: *count = L->out; return L->db;
        default: return NULL;
    }
}

lo_layer* lo_layer_new(size_t in, size_t out) {
    lo_layer* L = calloc(1, sizeof(lo_layer));
    if (!L || lo_layer_init(L, in, out)) {
        free(L);
        return NULL;
    }
    return L;
}

void lo_layer_delete(lo_layer* L) {
    if (!L) return;
    lo_layer_free(L);
    free(L);
}
