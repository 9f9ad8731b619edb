// layer_kernels.cuh -- per-layer sm_100a kernels behind the reference's layer
// API (FullyConnectedLayer / SoftmaxOutputLayer forward+backward,
// LayerState::apply_updates).  Row-major weights W[i*O + o]
// (include/lane/layers.hpp:78-80).  STRICT kernels follow the reference's
// evaluation order and rounding exactly; FAST kernels reassociate sums.
#pragma once

#include "common.cuh"

namespace lane_b200 {

enum Act : int { ACT_NONE = 0, ACT_TANH = 1 };

// ---------------------------------------------------------------------------
// netin (layers.cpp:27-41) + activation (layers.cpp:43-49).
// STRICT: one thread per output j, i ascending, mul then add (2 roundings).
// Threads of a warp read consecutive j of the same row i -> coalesced.
// x_src may differ from `inputs`; block 0 then caches x into `inputs`
// (compute_netin's `inputs = input`).
__global__ void k_netin_strict(const float* __restrict__ x_src, float* __restrict__ inputs,
                               const float* __restrict__ W, const float* __restrict__ b,
                               float* __restrict__ z, float* __restrict__ a, int I, int O,
                               int act) {
    if (x_src != inputs && blockIdx.x == 0)
        for (int i = threadIdx.x; i < I; i += blockDim.x) inputs[i] = x_src[i];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= O) return;
    float sum = 0.0f;
    for (int i = 0; i < I; ++i) sum = sadd(sum, smul(x_src[i], W[(size_t)i * O + j]));
    const float zj = sadd(sum, b[j]);
    z[j] = zj;
    if (act == ACT_TANH) a[j] = lane_libm::tanhf(zj);
}

// FAST netin, pass 1: split-K partial sums.  Block (32, 8): lane -> column j
// (coalesced 128 B row segments), warp row -> interleaved i; blockIdx.y -> a
// contiguous K chunk.  part[s*O + j] = partial over chunk s.
__global__ void k_netin_fast_part(const float* __restrict__ x, const float* __restrict__ W,
                                  float* __restrict__ part, int I, int O, int chunk) {
    __shared__ float red[8][33];
    const int j = blockIdx.x * 32 + threadIdx.x;
    const int i0 = blockIdx.y * chunk, i1 = min(I, i0 + chunk);
    float acc = 0.0f;
    if (j < O)
        for (int i = i0 + threadIdx.y; i < i1; i += 8) acc = fmaf(x[i], W[(size_t)i * O + j], acc);
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && j < O) {
        float s = red[0][threadIdx.x];
#pragma unroll
        for (int r = 1; r < 8; ++r) s += red[r][threadIdx.x];
        part[(size_t)blockIdx.y * O + j] = s;
    }
}

// FAST netin, pass 2: fixed-order sum of the S partials + bias + activation.
__global__ void k_netin_fast_finish(const float* __restrict__ part, int S,
                                    const float* __restrict__ x_src, float* __restrict__ inputs,
                                    int I, const float* __restrict__ b, float* __restrict__ z,
                                    float* __restrict__ a, int O, int act) {
    if (x_src != inputs && blockIdx.x == 0)
        for (int i = threadIdx.x; i < I; i += blockDim.x) inputs[i] = x_src[i];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= O) return;
    float s = 0.0f;
    for (int k = 0; k < S; ++k) s += part[(size_t)k * O + j];
    const float zj = s + b[j];
    z[j] = zj;
    if (act == ACT_TANH) a[j] = lane_libm::tanhf(zj);
}

// Softmax over netin (layers.cpp:71-87), one block.  STRICT: sequential max
// and sum on thread 0, exactly the reference order.  FAST: block tree.
__global__ void k_softmax(const float* __restrict__ z, float* __restrict__ p, int O, int strict) {
    __shared__ float sh_max, sh_sum;
    __shared__ float wred[32];
    const int t = threadIdx.x, nt = blockDim.x;
    if (strict) {
        if (t == 0) {
            float m = z[0];
            for (int j = 1; j < O; ++j) m = ref_max(m, z[j]);
            sh_max = m;
        }
        __syncthreads();
        for (int j = t; j < O; j += nt) p[j] = lane_libm::expf(ssub(z[j], sh_max));
        __syncthreads();
        if (t == 0) {
            float s = 0.0f;
            for (int j = 0; j < O; ++j) s = sadd(s, p[j]);
            sh_sum = s;
        }
        __syncthreads();
        for (int j = t; j < O; j += nt) p[j] = __fdiv_rn(p[j], sh_sum);
        return;
    }
    float m = -INFINITY;
    for (int j = t; j < O; j += nt) m = fmaxf(m, z[j]);
    m = warp_max(m);
    if ((t & 31) == 0) wred[t >> 5] = m;
    __syncthreads();
    if (t < 32) {
        float v = t < (nt + 31) / 32 ? wred[t] : -INFINITY;
        v = warp_max(v);
        if (t == 0) sh_max = v;
    }
    __syncthreads();
    float s = 0.0f;
    for (int j = t; j < O; j += nt) {
        const float e = lane_libm::expf(z[j] - sh_max);
        p[j] = e;
        s += e;
    }
    s = warp_sum(s);
    __syncthreads();
    if ((t & 31) == 0) wred[t >> 5] = s;
    __syncthreads();
    if (t < 32) {
        float v = t < (nt + 31) / 32 ? wred[t] : 0.0f;
        v = warp_sum(v);
        if (t == 0) sh_sum = v;
    }
    __syncthreads();
    for (int j = t; j < O; j += nt) p[j] = __fdiv_rn(p[j], sh_sum);
}

// ---------------------------------------------------------------------------
// Deltas.  softmax_backward_tuple (layers.hpp:33): delta = p - t;
// delta_biases = -eta * delta (layers.hpp:39).
__global__ void k_delta_softmax(const float* __restrict__ p, const float* __restrict__ t,
                                float* __restrict__ d, float* __restrict__ db, float neg_eta,
                                int O) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= O) return;
    const float delta = ssub(p[o], t[o]);
    d[o] = delta;
    db[o] = smul(neg_eta, delta);
}

// fc_backward_tuple (layers.hpp:49-53): s_o = sum_{k asc} nd[k]*nW[o*N + k];
// delta = (1 - a_o*a_o) * s_o.  STRICT: thread per o, sequential.
__global__ void k_delta_fc_strict(const float* __restrict__ a, const float* __restrict__ nW,
                                  const float* __restrict__ nd, float* __restrict__ d,
                                  float* __restrict__ db, float neg_eta, int O, int N) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= O) return;
    float s = 0.0f;
    const float* row = nW + (size_t)o * N;
    for (int k = 0; k < N; ++k) s = sadd(s, smul(nd[k], row[k]));
    const float delta = tanh_grad(a[o], s);
    d[o] = delta;
    db[o] = smul(neg_eta, delta);
}

// FAST: one warp per o, lanes stride the (contiguous) row, shuffle tree.
__global__ void k_delta_fc_fast(const float* __restrict__ a, const float* __restrict__ nW,
                                const float* __restrict__ nd, float* __restrict__ d,
                                float* __restrict__ db, float neg_eta, int O, int N) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= O) return;
    const float* row = nW + (size_t)warp * N;
    float s = 0.0f;
    for (int k = lane; k < N; k += 32) s = fmaf(nd[k], row[k], s);
    s = warp_sum(s);
    if (lane == 0) {
        const float delta = tanh_grad(a[warp], s);
        d[warp] = delta;
        db[warp] = smul(neg_eta, delta);
    }
}

// Outer product: G[i][o] = delta_o * x_i ; DW[i][o] = -eta * G[i][o]
// (layers.hpp:34-35, :54-56).  Element-wise, rounding identical to the
// reference in both modes.  Grid-stride over I*O, o fastest (coalesced).
__global__ void k_outer(const float* __restrict__ d, const float* __restrict__ x,
                        float* __restrict__ G, float* __restrict__ DW, float neg_eta, int I,
                        int O) {
    const size_t n = (size_t)I * O;
    if (n <= 0xffffffffull) {  // 32-bit index math (no 64-bit division per element)
        const unsigned un = (unsigned)n, uO = (unsigned)O;
        for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < un; e += gridDim.x * blockDim.x) {
            const unsigned i = e / uO, o = e - i * uO;
            const float g = smul(d[o], x[i]);
            G[e] = g;
            DW[e] = smul(neg_eta, g);
        }
        return;
    }
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / O), o = (int)(e - (size_t)i * O);
        const float g = smul(d[o], x[i]);
        G[e] = g;
        DW[e] = smul(neg_eta, g);
    }
}

// Same with O % 4 == 0: threads own a column quad (the delta quad stays in
// registers) and walk rows with stride gridDim.y; float4 streaming stores.
// HBM-bound: 8 B written per element.
__global__ void __launch_bounds__(256) k_outer4(const float4* __restrict__ d, const float* __restrict__ x,
                                                float4* __restrict__ G, float4* __restrict__ DW, float neg_eta,
                                                int I, int Q) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Q) return;
    const float4 dq = d[q];
    for (int i = blockIdx.y; i < I; i += gridDim.y) {
        const float xi = x[i];
        float4 g;
        g.x = smul(dq.x, xi);
        g.y = smul(dq.y, xi);
        g.z = smul(dq.z, xi);
        g.w = smul(dq.w, xi);
        const size_t e = (size_t)i * Q + q;
        __stcs(G + e, g);
        __stcs(DW + e, make_float4(smul(neg_eta, g.x), smul(neg_eta, g.y), smul(neg_eta, g.z), smul(neg_eta, g.w)));
    }
}

// LayerState::apply_updates (layers.cpp:18-25): W += DW ; b += db.
__global__ void k_apply_updates(float* __restrict__ W, const float* __restrict__ DW, size_t n,
                                float* __restrict__ b, const float* __restrict__ db, int O) {
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(DW)) & 15) == 0;
    if (vec) {
        const size_t n4 = n / 4;
        float4* W4 = reinterpret_cast<float4*>(W);
        const float4* D4 = reinterpret_cast<const float4*>(DW);
        for (size_t e = tid; e < n4; e += stride) {
            float4 w = W4[e];
            const float4 dw = D4[e];
            w.x = sadd(w.x, dw.x);
            w.y = sadd(w.y, dw.y);
            w.z = sadd(w.z, dw.z);
            w.w = sadd(w.w, dw.w);
            W4[e] = w;
        }
        for (size_t e = n4 * 4 + tid; e < n; e += stride) W[e] = sadd(W[e], DW[e]);
    } else {
        for (size_t e = tid; e < n; e += stride) W[e] = sadd(W[e], DW[e]);
    }
    for (size_t j = tid; j < (size_t)O; j += stride) b[j] = sadd(b[j], db[j]);
}

// cross_entropy (network.cpp:68-79) and argmax (network.cpp:13-21) of one
// sample, accumulated like train(): loss_sum (double) += ce ; correct += hit.
__global__ void k_loss_accumulate(const float* __restrict__ p, const float* __restrict__ t,
                                  int O, double* loss_sum, unsigned long long* correct) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    float loss = 0.0f;
    int bp = 0, bt = 0;
    for (int o = 0; o < O; ++o) {
        if (t[o] != 0.0f) {
            const float q = p[o] < 1e-12f ? 1e-12f : p[o];
            loss = ssub(loss, smul(t[o], lane_libm::logf(q)));
        }
        if (o > 0 && p[o] > p[bp]) bp = o;
        if (o > 0 && t[o] > t[bt]) bt = o;
    }
    if (loss_sum) *loss_sum = __dadd_rn(*loss_sum, (double)loss);
    if (correct) *correct += (bp == bt) ? 1ull : 0ull;
}

// Copies sample k = order[*step] (or *step mod n) into the first layer's
// inputs and the target staging buffer, then advances *step when `advance`.
__global__ void k_stage_sample(const float* __restrict__ X, const float* __restrict__ T,
                               const uint32_t* __restrict__ order, long long n,
                               long long* step, float* __restrict__ x_dst, int I,
                               float* __restrict__ t_dst, int C) {
    const long long s = *step;
    const long long k = order ? (long long)order[s] : s % n;
    for (int i = threadIdx.x; i < I; i += blockDim.x) x_dst[i] = X[k * I + i];
    for (int c = threadIdx.x; c < C; c += blockDim.x) t_dst[c] = T[k * C + c];
}

__global__ void k_step_advance(long long* step) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *step += 1;
}

}  // namespace lane_b200
