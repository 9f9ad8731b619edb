// sgd_tiny.cuh -- online SGD (batch 1) for tiny one-hidden-layer networks
// (input, hidden <= 32, classes <= 16: the reference's Iris 4-8-3 acceptance
// net, XOR 2-4-2), ONE warp for the whole stream.
//
// For these sizes the windowed kernel (sgd_window.cuh) is all fixed cost:
// ~1,200 cycles per sample of chain, helper and producer protocol for a few
// dozen FLOPs.  Here lane j owns hidden unit j -- its W0 column and W1 row in
// registers -- and lane k owns class k with a copy of W1's column k (both
// copies receive the identical update, so they stay bit-equal).  A sample is
// a handful of shuffles between the lanes:
//   x_i -> all; z0_j, a0_j (lane j); a_j -> all; z1_k (lane k, j ascending);
//   z1 -> all for the max; e_k (lane k) -> all for the sum; p_k, d1_k;
//   d1 -> all; d0_j (lane j, k ascending); the updates.
// The arithmetic is the reference's exactly -- every sum in the reference's
// order, separately rounded mul / add (smul / sadd), the glibc tanhf / expf /
// logf restatements, __fdiv_rn -- so the kernel runs STRICT numerics
// bit-for-bit (network.cpp:164-170 -> BackwardPlan::run, layers.hpp:28-61,
// layers.cpp:18-49, :71-87, network.cpp:68-79): the STRICT stream of these
// nets, which otherwise runs the per-sample layer kernels, becomes one
// launch.  (FAST stays on the windowed kernel: a one-warp chain with FMA
// sums and libdevice transcendentals measured 1.1-1.6M samples/s at C1
// against the window kernel's 1.58M.)
// The last sample's LayerState vectors, gradients and delta weights are
// written at the end, as BackwardPlan::run leaves them.
#pragma once

#include "common.cuh"

namespace lane_b200 {

constexpr int kTinyMaxI = 32, kTinyMaxH = 32, kTinyMaxC = 16;

struct TinyArgs {
    int I, H, C;
    const float* X;
    const float* T;
    const uint32_t* order;  // stream position -> row (nullptr: (base + s) mod n)
    long long n, n_steps, base;
    float neg_eta;
    float *W0, *b0, *W1, *b1;                    // parameters, updated in place
    float *x0, *z0, *a0, *d0, *db0, *G0, *DW0;   // layer 0 LayerState (last sample)
    float *x1, *z1, *a1, *d1, *db1, *G1, *DW1;   // layer 1 (output) LayerState
    double* loss_sum;                            // += cross entropy per sample (double, in order)
    unsigned long long* correct;                 // += argmax hits
};

template <int IM, int HM, int CM>
__global__ void __launch_bounds__(32, 1) k_sgd_tiny(TinyArgs A) {
    const int lane = threadIdx.x;
    const int I = A.I, H = A.H, C = A.C;
    const bool hj = lane < H, ck = lane < C;
    const float neg_eta = A.neg_eta;
    float w0[IM], w1r[CM], w1c[HM];
#pragma unroll
    for (int i = 0; i < IM; ++i) w0[i] = (hj && i < I) ? A.W0[(size_t)i * H + lane] : 0.0f;
#pragma unroll
    for (int k = 0; k < CM; ++k) w1r[k] = (hj && k < C) ? A.W1[(size_t)lane * C + k] : 0.0f;
#pragma unroll
    for (int j = 0; j < HM; ++j) w1c[j] = (ck && j < H) ? A.W1[(size_t)j * C + lane] : 0.0f;
    float b0 = hj ? A.b0[lane] : 0.0f;
    float b1 = ck ? A.b1[lane] : 0.0f;
    double lacc = (lane == 0 && A.loss_sum) ? *A.loss_sum : 0.0;
    unsigned long long hits = 0;
    // stream position -> row: order[s], or (base + s) mod n kept incrementally
    // (no 64-bit division per sample)
    long long seq = A.n > 0 ? A.base % A.n : 0;
    auto row = [&](long long s) -> long long {
        if (A.order) return (long long)A.order[s];
        const long long r = seq;
        if (++seq == A.n) seq = 0;
        return r;
    };
    // the current and next samples' x (lane i) and t (lane k)
    float xn = 0.0f, tn = 0.0f;
    if (A.n_steps > 0) {
        const long long r = row(0);
        xn = lane < I ? A.X[r * I + lane] : 0.0f;
        tn = ck ? A.T[r * C + lane] : 0.0f;
    }
    float xv = 0.0f, tv = 0.0f, z0 = 0.0f, a0 = 0.0f, d0 = 0.0f, z1 = 0.0f, p = 0.0f, d1 = 0.0f;
    float x_all[IM], a_all[HM], d1_all[CM];
    for (long long s = 0; s < A.n_steps; ++s) {
        xv = xn;
        tv = tn;
        if (s + 1 < A.n_steps) {
            const long long r = row(s + 1);
            xn = lane < I ? __ldg(A.X + r * I + lane) : 0.0f;
            tn = ck ? __ldg(A.T + r * C + lane) : 0.0f;
        }
        // ---- forward, hidden layer (layers.cpp:27-49): i ascending
#pragma unroll
        for (int i = 0; i < IM; ++i) x_all[i] = __shfl_sync(0xffffffffu, xv, i);
        float sum = 0.0f;
#pragma unroll
        for (int i = 0; i < IM; ++i)
            if (i < I) sum = sadd(sum, smul(x_all[i], w0[i]));
        z0 = sadd(sum, b0);
        a0 = lane_libm::tanhf(z0);
        // ---- forward, softmax layer (layers.cpp:71-87): j ascending, then the
        //      max, the exponentials and their sum in class order
#pragma unroll
        for (int j = 0; j < HM; ++j) a_all[j] = __shfl_sync(0xffffffffu, a0, j);
        float s1 = 0.0f;
#pragma unroll
        for (int j = 0; j < HM; ++j)
            if (j < H) s1 = sadd(s1, smul(a_all[j], w1c[j]));
        z1 = sadd(s1, b1);
        float m = __shfl_sync(0xffffffffu, z1, 0);
#pragma unroll
        for (int k = 1; k < CM; ++k) {
            const float zk = __shfl_sync(0xffffffffu, z1, k);
            if (k < C) m = ref_max(m, zk);
        }
        const float e = lane_libm::expf(ssub(z1, m));
        float es = 0.0f;
#pragma unroll
        for (int k = 0; k < CM; ++k) {
            const float ek = __shfl_sync(0xffffffffu, e, k);
            if (k < C) es = sadd(es, ek);
        }
        p = __fdiv_rn(e, es);
        // ---- backward (layers.hpp:28-61): d1 = p - t; d0 with the pre-update W1
        d1 = ssub(p, tv);
#pragma unroll
        for (int k = 0; k < CM; ++k) d1_all[k] = __shfl_sync(0xffffffffu, d1, k);
        float s0 = 0.0f;
#pragma unroll
        for (int k = 0; k < CM; ++k)
            if (k < C) s0 = sadd(s0, smul(d1_all[k], w1r[k]));
        d0 = tanh_grad(a0, s0);
        // ---- apply_updates (layers.cpp:18-25): w + (-eta * (delta * x))
#pragma unroll
        for (int i = 0; i < IM; ++i)
            if (i < I) w0[i] = sgd_apply(w0[i], neg_eta, d0, x_all[i]);
        b0 = sadd(b0, smul(neg_eta, d0));
#pragma unroll
        for (int k = 0; k < CM; ++k)
            if (k < C) w1r[k] = sgd_apply(w1r[k], neg_eta, d1_all[k], a0);
#pragma unroll
        for (int j = 0; j < HM; ++j)
            if (j < H) w1c[j] = sgd_apply(w1c[j], neg_eta, d1, a_all[j]);
        b1 = sadd(b1, smul(neg_eta, d1));
        // ---- cross entropy + argmax (network.cpp:13-21, :68-79), in class order
        {
            float loss = 0.0f, pb = 0.0f, tb = 0.0f;
            int bp = 0, bt = 0;
#pragma unroll
            for (int k = 0; k < CM; ++k) {
                const float pk = __shfl_sync(0xffffffffu, p, k);
                const float tk = __shfl_sync(0xffffffffu, tv, k);
                if (k < C && lane == 0) {
                    if (tk != 0.0f) loss = ssub(loss, smul(tk, lane_libm::logf(pk < 1e-12f ? 1e-12f : pk)));
                    if (k == 0 || pk > pb) {
                        pb = pk;
                        bp = k;
                    }
                    if (k == 0 || tk > tb) {
                        tb = tk;
                        bt = k;
                    }
                }
            }
            if (lane == 0) {
                lacc = __dadd_rn(lacc, (double)loss);
                hits += bp == bt ? 1ull : 0ull;
            }
        }
    }
    if (A.n_steps == 0) return;
    // ---- write back: parameters and the last sample's LayerState
    // (compile-time loop bounds: a runtime-indexed register array would be
    // demoted to local memory for the whole kernel)
    if (hj) {
#pragma unroll
        for (int i = 0; i < IM; ++i) {
            if (i >= I) break;
            A.W0[(size_t)i * H + lane] = w0[i];
            const float g = smul(d0, x_all[i]);
            A.G0[(size_t)i * H + lane] = g;
            A.DW0[(size_t)i * H + lane] = smul(neg_eta, g);
        }
#pragma unroll
        for (int k = 0; k < CM; ++k) {
            if (k >= C) break;
            A.W1[(size_t)lane * C + k] = w1r[k];
            const float g = smul(d1_all[k], a0);
            A.G1[(size_t)lane * C + k] = g;
            A.DW1[(size_t)lane * C + k] = smul(neg_eta, g);
        }
        A.b0[lane] = b0;
        A.z0[lane] = z0;
        A.a0[lane] = a0;
        A.d0[lane] = d0;
        A.db0[lane] = smul(neg_eta, d0);
        A.x1[lane] = a0;
    }
    if (lane < I) A.x0[lane] = xv;
    if (ck) {
        A.b1[lane] = b1;
        A.z1[lane] = z1;
        A.a1[lane] = p;
        A.d1[lane] = d1;
        A.db1[lane] = smul(neg_eta, d1);
    }
    if (lane == 0) {
        if (A.loss_sum) *A.loss_sum = lacc;
        if (A.correct) *A.correct += hits;
    }
}

inline bool tiny_fits(int I, int H, int C) {
    return I >= 1 && I <= kTinyMaxI && H >= 1 && H <= kTinyMaxH && C >= 1 && C <= kTinyMaxC;
}

inline void tiny_launch(cudaStream_t st, const TinyArgs& A) {
    if (A.I <= 8 && A.H <= 8 && A.C <= 4)
        k_sgd_tiny<8, 8, 4><<<1, 32, 0, st>>>(A);
    else
        k_sgd_tiny<kTinyMaxI, kTinyMaxH, kTinyMaxC><<<1, 32, 0, st>>>(A);
}

}  // namespace lane_b200
