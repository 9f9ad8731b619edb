// minibatch.cuh -- the mini-batch / momentum / data-parallel extension
// (SURVEY.md 8a row a15, 8e).  Not in the reference; defined so
// that B=1, mu=0 reduces to BackwardPlan::run (oracle/lane_oracle.c
// lo_minibatch_step):
//     G  = (1/B_global) * sum_b delta_b (x) x_b
//     DW = mu*DW + (-eta)*G   (DW = (-eta)*G when mu == 0)
//     W += DW ;  biases likewise.
// Per layer the step is three GEMMs -- forward Z = X W (+b, tanh), dgrad
// S = D' W'^T (x tanh'), wgrad G = X^T D -- plus a row softmax and the update.
// Data parallel: each rank runs its local batch; each layer's span of the flat
// gradient-sum buffer (G and bias sums, contiguous per layer) is summed with an
// NCCL fp32 allreduce as soon as that layer's wgrad is done (one per layer, in
// reverse layer order, overlapping the rest of the backward), then every rank
// applies the identical update.
#pragma once

#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"
#include "nvls.cuh"

namespace lane_b200 {

#define LANE_NCCL(call)                                                                   \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess)                                                            \
            throw ::lane_b200::Error(LANE_ERR_NCCL, std::string(#call) + ": " +           \
                                                        ncclGetErrorString(r_));          \
    } while (0)

struct MinibatchComm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

struct MinibatchState {
    float* ws = nullptr;  // GEMM workspace (split-K partials / 3xTF32 splits)
    size_t ws_count = 0;
    uint64_t ws_gen = 0;  // reallocation count: part of the captured step graph's key
    int* counters = nullptr;  // stream-K tile counters of the persistent GEMM
    size_t counters_count = 0;
    cudaStream_t comm_stream = nullptr;  // per-layer gradient allreduces (data parallel)
    std::vector<cudaEvent_t> ev;         // one per layer + the join
    unsigned* stats = nullptr;           // 3xF16 operand maxima (MbStats)
    size_t stats_count = 0;
};

inline void minibatch_free(MinibatchState& s) {
    if (s.ws) cudaFree(s.ws);
    s.ws = nullptr;
    s.ws_count = 0;
    if (s.counters) cudaFree(s.counters);
    s.counters = nullptr;
    s.counters_count = 0;
    if (s.stats) cudaFree(s.stats);
    s.stats = nullptr;
    s.stats_count = 0;
    for (cudaEvent_t e : s.ev) cudaEventDestroy(e);
    s.ev.clear();
    if (s.comm_stream) cudaStreamDestroy(s.comm_stream);
    s.comm_stream = nullptr;
}

inline void nccl_unique_id(void* out, size_t bytes) {
    if (!out || bytes < sizeof(ncclUniqueId)) throw Error(LANE_ERR_CONFIG, "unique id buffer too small");
    ncclUniqueId id;
    LANE_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
}

inline void comm_init(MinibatchComm& c, int rank, int world, const void* id, size_t bytes) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(LANE_ERR_CONFIG, "bad rank/world");
    if (!id || bytes < sizeof(ncclUniqueId)) throw Error(LANE_ERR_CONFIG, "bad unique id");
    if (c.comm) {
        ncclCommDestroy(c.comm);
        c.comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    LANE_NCCL(ncclCommInitRank(&c.comm, world, uid, rank));
    c.rank = rank;
    c.world = world;
}

inline void comm_destroy(MinibatchComm& c) {
    if (c.comm) ncclCommDestroy(c.comm);
    c.comm = nullptr;
    c.rank = 0;
    c.world = 1;
}

inline void allreduce_grads(MinibatchComm& c, float* grads, size_t count, cudaStream_t stream) {
    if (!c.comm || c.world == 1) return;
    LANE_NCCL(ncclAllReduce(grads, grads, count, ncclFloat32, ncclSum, c.comm, stream));
}

// ------------------------------------------------------------- kernels ---

// Row softmax + output deltas + cross entropy for a batch (one warp per row,
// C <= 128): P = softmax(Z + b) (Z already has the bias), D = P - T,
// loss_sum += sum_rows CE (double, row order via a serial final pass).
__global__ void k_softmax_rows(const float* __restrict__ Z, float* __restrict__ P,
                               const float* __restrict__ T, float* __restrict__ D,
                               float* __restrict__ row_loss, int B, int C) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= B) return;
    const float* z = Z + (size_t)warp * C;
    const float* t = T + (size_t)warp * C;
    float e[4];
    float m = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        if (k < C) m = fmaxf(m, z[k]);
    }
    m = warp_max(m);
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        e[q] = k < C ? lane_libm::expf(ssub(z[k], m)) : 0.0f;
        s += e[q];
    }
    s = warp_sum(s);
    float loss = 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        if (k < C) {
            const float p = __fdiv_rn(e[q], s);
            P[(size_t)warp * C + k] = p;
            D[(size_t)warp * C + k] = ssub(p, t[k]);
            if (t[k] != 0.0f) loss = sadd(loss, smul(t[k], lane_libm::logf(p < 1e-12f ? 1e-12f : p)));
        }
    }
    loss = warp_sum(loss);
    if (lane == 0 && row_loss) row_loss[warp] = -loss;
}

// loss_sum += sum_b row_loss[b] in double: lane l sums rows l, l+32, ... in
// order, then a fixed butterfly (deterministic, one warp)
__global__ void k_loss_rows(const float* __restrict__ row_loss, int B, double* loss_sum) {
    if (blockIdx.x != 0 || threadIdx.x >= 32 || !loss_sum) return;
    double s = 0.0;
    for (int b = threadIdx.x; b < B; b += 32) s += (double)row_loss[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *loss_sum += s;
}

// evaluate() over a batch of rows (FAST numerics): thread per row, the
// softmax of the logits Z (bias included) and k_loss_accumulate's per-sample
// cross entropy and argmax test (ties to the lowest index, network.cpp:13-21).
__global__ void k_eval_rows(const float* __restrict__ Z, const float* __restrict__ T, int B, int C,
                            float* __restrict__ row_loss, float* __restrict__ row_ok) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const float* z = Z + (size_t)b * C;
    const float* t = T + (size_t)b * C;
    float m = z[0];
    for (int k = 1; k < C; ++k) m = fmaxf(m, z[k]);
    float s = 0.0f;
    for (int k = 0; k < C; ++k) s += lane_libm::expf(ssub(z[k], m));
    float loss = 0.0f;
    int bp = 0, bt = 0;
    float pbest = -1.0f;
    for (int k = 0; k < C; ++k) {
        const float p = __fdiv_rn(lane_libm::expf(ssub(z[k], m)), s);
        if (t[k] != 0.0f) loss = ssub(loss, smul(t[k], lane_libm::logf(p < 1e-12f ? 1e-12f : p)));
        if (k == 0 || p > pbest) {
            pbest = p;
            bp = k;
        }
        if (k > 0 && t[k] > t[bt]) bt = k;
    }
    row_loss[b] = loss;
    row_ok[b] = bp == bt ? 1.0f : 0.0f;
}

// loss_sum += sum_b row_loss[b] (double; lane-strided then a fixed butterfly),
// correct += sum_b row_ok[b]
__global__ void k_eval_reduce(const float* __restrict__ row_loss, const float* __restrict__ row_ok, int B,
                              double* loss_sum, unsigned long long* correct) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    double s = 0.0;
    unsigned long long ok = 0;
    for (int b = threadIdx.x; b < B; b += 32) {
        s += (double)row_loss[b];
        ok += row_ok[b] != 0.0f ? 1ull : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        ok += __shfl_xor_sync(0xffffffffu, ok, o);
    }
    if (threadIdx.x == 0) {
        *loss_sum += s;
        *correct += ok;
    }
}

// Momentum SGD on a flat range: g = gsum * invB; DW = mu*DW + (-eta)*g;
// W += DW.  Writes the mean gradient back to gsum (LANE_BUF_G semantics).
// the whole parameter set in one pass: params, grads and velocities share one
// arena layout (W_0 | b_0 | W_1 | ...; 256-byte pieces, zero padding), so
// element e of each region belongs to the same parameter.  16-byte accesses.
__global__ void k_momentum_update_all(float4* __restrict__ W, float4* __restrict__ DW,
                                      float4* __restrict__ gsum, size_t n4, float invB, float neg_eta,
                                      float mu) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4;
         e += (size_t)gridDim.x * blockDim.x) {
        // plain SGD (mu == 0) never reads the old delta_weights
        float4 g = gsum[e], v = mu == 0.0f ? make_float4(0.f, 0.f, 0.f, 0.f) : DW[e], w = W[e];
        float* gp = &g.x;
        float* vp = &v.x;
        float* wp = &w.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float gi = smul(gp[i], invB);
            gp[i] = gi;
            const float step = smul(neg_eta, gi);
            vp[i] = mu == 0.0f ? step : sadd(smul(mu, vp[i]), step);
            wp[i] = sadd(wp[i], vp[i]);
        }
        gsum[e] = g;
        DW[e] = v;
        W[e] = w;
    }
}

// The same update over a list of spans of the arena (float4 offsets from the
// region bases): the pieces a fused wgrad + update epilogue did not cover.
constexpr int kMaxUpdSpans = 32;
struct UpdSpans {
    int n = 0;
    unsigned long long beg[kMaxUpdSpans], end[kMaxUpdSpans];
};
template <bool PRESCALED>
__global__ void k_momentum_update_spans(float4* __restrict__ W, float4* __restrict__ DW, float4* __restrict__ gsum,
                                        UpdSpans sp, unsigned long long total, float invB, float neg_eta, float mu) {
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long e = t;
        int k = 0;
        while (k < sp.n - 1 && e >= sp.end[k] - sp.beg[k]) {
            e -= sp.end[k] - sp.beg[k];
            ++k;
        }
        e += sp.beg[k];
        float4 g = gsum[e], v = mu == 0.0f ? make_float4(0.f, 0.f, 0.f, 0.f) : DW[e], w = W[e];
        float* gp = &g.x;
        float* vp = &v.x;
        float* wp = &w.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            // PRESCALED: gsum already holds g = sum * invB (the wgrad epilogue's)
            const float gi = PRESCALED ? gp[i] : smul(gp[i], invB);
            gp[i] = gi;
            const float step = smul(neg_eta, gi);
            vp[i] = mu == 0.0f ? step : sadd(smul(mu, vp[i]), step);
            wp[i] = sadd(wp[i], vp[i]);
        }
        if (!PRESCALED) gsum[e] = g;
        DW[e] = v;
        W[e] = w;
    }
}

__global__ void k_momentum_update(float* __restrict__ W, float* __restrict__ DW,
                                  float* __restrict__ gsum, size_t n, float invB, float neg_eta,
                                  float mu) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
        const float g = smul(gsum[e], invB);
        gsum[e] = g;
        const float step = smul(neg_eta, g);
        const float dw = mu == 0.0f ? step : sadd(smul(mu, DW[e]), step);
        DW[e] = dw;
        W[e] = sadd(W[e], dw);
    }
}

// --------------------------------------------------------------- driver ---

// Stage a batch: the first layer's inputs (LayerState::inputs) and the
// targets, device to device.  Kept out of the captured step graph so the graph
// only ever touches the network's own buffers.
template <class Ctx, class Net>
void minibatch_stage(Ctx& c, Net& net, const float* X, const float* T, size_t Bsz) {
    if (net.classes > 128) throw Error(LANE_ERR_CONFIG, "minibatch: classes must be <= 128");
    LANE_CUDA(cudaMemcpyAsync(net.L(0).buf[LANE_BUF_INPUTS], X, Bsz * net.input_width * sizeof(float),
                              cudaMemcpyDeviceToDevice, c.stream));
    LANE_CUDA(cudaMemcpyAsync(net.target_stage, T, Bsz * net.classes * sizeof(float), cudaMemcpyDeviceToDevice,
                              c.stream));
}

// Forward, softmax/CE and the backward of a staged batch: per layer l the
// gradient sums G_l = X_l^T D_l and gb_l = colsum(D_l) land in the grads arena
// (sums over the local rows, not yet divided by B).  The backward runs in
// reverse layer order with each layer's wgrad issued before the next dgrad, so
// in data-parallel mode (`allreduce`) layer l's span of the arena goes to NCCL
// on the communication stream right after its wgrad and overlaps every
// remaining dgrad and wgrad; the compute stream joins the communication stream
// at the end.  Capturable in a CUDA graph.
// Operand maxima of the 3xF16 GEMMs (gemm_h3.cuh), per layer l with input
// width I and output width O: rows / columns of the layer input act_l (B, I),
// of W_l (I, O) and of the layer's output deltas D_l (B, O).  Produced once per
// step -- W_l and act_0 by one pass each, act_{l+1} and D_{l-1} by the
// epilogues of the GEMMs that write them -- instead of two passes per GEMM.
struct MbStats {
    std::vector<unsigned*> act_row, act_col, w_row, w_col, d_row, d_col;
};

template <class Net>
MbStats minibatch_stats(Net& net, size_t B, GemmCtx& g, cudaStream_t st) {
    const int nl = static_cast<int>(net.layers.size());
    size_t need = 0;
    for (int l = 0; l < nl; ++l) need += 2 * B + 2 * net.L(l).I + 2 * net.L(l).O;
    auto& M = net.mb;
    if (M.stats_count < need) {
        if (M.stats) LANE_CUDA(cudaFree(M.stats));
        LANE_CUDA(cudaMalloc(reinterpret_cast<void**>(&M.stats), need * sizeof(unsigned)));
        M.stats_count = need;
        ++M.ws_gen;  // captured step graphs hold the old pointer
    }
    (void)g;
    LANE_CUDA(cudaMemsetAsync(M.stats, 0, need * sizeof(unsigned), st));
    MbStats S;
    unsigned* p = M.stats;
    for (int l = 0; l < nl; ++l) {
        const size_t I = net.L(l).I, O = net.L(l).O;
        S.act_row.push_back(p), p += B;
        S.act_col.push_back(p), p += I;
        S.w_row.push_back(p), p += I;
        S.w_col.push_back(p), p += O;
        S.d_row.push_back(p), p += B;
        S.d_col.push_back(p), p += O;
    }
    return S;
}

struct FusedUpdate {
    float inv_b, eta, mu;
    bool fused_w[kMaxUpdSpans];   // out: layer l's weights were updated by its wgrad epilogue
    bool scaled_g[kMaxUpdSpans];  // out: layer l's G already holds the mean (3xF16 wgrad epilogue)
};

template <class Ctx, class Net>
void minibatch_grads_body(Ctx& c, Net& net, size_t Bsz, double* loss_sum, bool allreduce,
                          FusedUpdate* fused = nullptr) {
    const int B = static_cast<int>(Bsz);
    const int nl = static_cast<int>(net.layers.size());
    const int C = static_cast<int>(net.classes);
    cudaStream_t st = c.stream;
    GemmCtx g{c.stream,   c.sm_count,        &net.mb.ws,       &net.mb.ws_count, &c.launches,
              &net.mb.ws_gen, &net.mb.counters, &net.mb.counters_count};
    // which GEMMs run on the 3xF16 kernel, and so which operand maxima exist
    auto input = [&](int l) {
        return l == 0 ? net.L(0).buf[LANE_BUF_INPUTS] : net.L(l - 1).buf[LANE_BUF_OUTPUTS];
    };
    auto fwd_h3 = [&](int l) {
        auto& Ly = net.L(l);
        return gemm_will_h3(GemmOp::NN, B, (int)Ly.O, (int)Ly.I, input(l), (int)Ly.I, Ly.buf[LANE_BUF_W], (int)Ly.O,
                            Ly.buf[LANE_BUF_NETIN]);
    };
    auto dgrad_h3 = [&](int l) {  // l >= 1: D_{l-1} = D_l W_l^T
        if (l < 1) return false;
        auto& Ly = net.L(l);
        auto& pv = net.L(l - 1);
        return gemm_will_h3(GemmOp::NT, B, (int)pv.O, (int)Ly.O, Ly.buf[LANE_BUF_DELTAS], (int)Ly.O,
                                      Ly.buf[LANE_BUF_W], (int)Ly.O, pv.buf[LANE_BUF_DELTAS]);
    };
    auto wgrad_h3 = [&](int l) {
        auto& Ly = net.L(l);
        return gemm_will_h3(GemmOp::TN, (int)Ly.I, (int)Ly.O, B, input(l), (int)Ly.I, Ly.buf[LANE_BUF_DELTAS],
                            (int)Ly.O, Ly.buf[LANE_BUF_G]);
    };
    bool any_h3 = false;
    for (int l = 0; l < nl; ++l) any_h3 = any_h3 || fwd_h3(l) || dgrad_h3(l) || wgrad_h3(l);
    MbStats S;
    if (any_h3) {
        S = minibatch_stats(net, Bsz, g, st);
        for (int l = 0; l < nl; ++l)
            if (fwd_h3(l) || dgrad_h3(l)) {
                absmax_rc_launch(st, net.L(l).buf[LANE_BUF_W], (int)net.L(l).I, (int)net.L(l).O, S.w_row[l],
                                 S.w_col[l]);
                c.launches += 1;
            }
        if (fwd_h3(0) || wgrad_h3(0)) {
            absmax_rc_launch(st, input(0), B, (int)net.L(0).I, S.act_row[0], S.act_col[0]);
            c.launches += 1;
        }
    }
    // forward
    for (int l = 0; l < nl; ++l) {
        auto& Ly = net.L(l);
        // layer l > 0 reads the previous layer's outputs in place (no copy)
        const float* in = input(l);
        const bool last = l == nl - 1;
        GemmMax mx;
        if (fwd_h3(l)) {
            mx.a = S.act_row[l];
            mx.b = S.w_col[l];
        }
        if (!last && (fwd_h3(l + 1) || wgrad_h3(l + 1))) {
            mx.orow = S.act_row[l + 1];
            mx.ocol = S.act_col[l + 1];
        }
        gemm(g, GemmOp::NN, B, (int)Ly.O, (int)Ly.I, in, (int)Ly.I, Ly.buf[LANE_BUF_W], (int)Ly.O,
             last ? Epi::BIAS : Epi::BIAS_TANH, Ly.buf[LANE_BUF_NETIN], Ly.buf[LANE_BUF_OUTPUTS],
             Ly.buf[LANE_BUF_B], nullptr, &mx);
    }
    auto& out = net.L(nl - 1);
    ensure_ws(g, (size_t)B);  // per-row losses live in the GEMM workspace between GEMMs
    k_softmax_rows<<<(B * 32 + 255) / 256, 256, 0, st>>>(out.buf[LANE_BUF_NETIN], out.buf[LANE_BUF_OUTPUTS],
                                                          net.target_stage, out.buf[LANE_BUF_DELTAS],
                                                          net.mb.ws, B, C);
    k_loss_rows<<<1, 32, 0, st>>>(net.mb.ws, B, loss_sum);
    c.launches += 2;
    auto& M = net.mb;
    if (allreduce) {
        if (!M.comm_stream) LANE_CUDA(cudaStreamCreateWithFlags(&M.comm_stream, cudaStreamNonBlocking));
        while ((int)M.ev.size() < nl + 1) {
            cudaEvent_t e;
            LANE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            M.ev.push_back(e);
        }
    }
    auto dgrad = [&](int l) {
        // dgrad with the pre-update weights: D_{l-1} = (D_l W_l^T) * (1 - A_{l-1}^2)
        auto& Ly = net.L(l);
        auto& pv = net.L(l - 1);
        GemmMax mx;
        if (dgrad_h3(l)) {
            mx.a = S.d_row[l];
            mx.b = S.w_row[l];
        }
        if (dgrad_h3(l - 1) || wgrad_h3(l - 1)) {
            mx.orow = S.d_row[l - 1];
            mx.ocol = S.d_col[l - 1];
        }
        gemm(g, GemmOp::NT, B, (int)pv.O, (int)Ly.O, Ly.buf[LANE_BUF_DELTAS], (int)Ly.O, Ly.buf[LANE_BUF_W],
             (int)Ly.O, Epi::TANH_GRAD, pv.buf[LANE_BUF_DELTAS], nullptr, nullptr, pv.buf[LANE_BUF_OUTPUTS], &mx);
    };
    auto wgrad_mx = [&](int l) {
        GemmMax mx;
        if (wgrad_h3(l)) {
            mx.a = S.act_col[l];
            mx.b = S.d_col[l];
        }
        return mx;
    };
    for (int l = nl - 1; l >= 0; --l) {
        auto& Ly = net.L(l);
        const float* in = l == 0 ? net.L(0).buf[LANE_BUF_INPUTS] : net.L(l - 1).buf[LANE_BUF_OUTPUTS];
        if (fused) {
            // one rank: the dgrad reads W_l first, then the wgrad's epilogue
            // updates W_l in place (G_l = X_l^T D_l / B, V_l, W_l)
            if (l > 0) dgrad(l);
            float* W = Ly.buf[LANE_BUF_W];
            float* V = Ly.buf[LANE_BUF_DW];
            fused->fused_w[l] = gemm_wgrad_update(g, (int)Ly.I, (int)Ly.O, B, in, Ly.buf[LANE_BUF_DELTAS],
                                                            Ly.buf[LANE_BUF_G], W, V, fused->inv_b, -fused->eta,
                                                            fused->mu);
            fused->scaled_g[l] = false;
            if (!fused->fused_w[l]) {
                GemmMax mx = wgrad_mx(l);
                // the 3xF16 wgrad stores the mean gradient directly (G = sum x 1/B,
                // the update's own first operation): the update pass then reads
                // G once and does not rewrite it -- 4 of its 20 bytes per weight
                if (wgrad_h3(l)) {
                    mx.out_scale = fused->inv_b;
                    fused->scaled_g[l] = true;
                }
                gemm(g, GemmOp::TN, (int)Ly.I, (int)Ly.O, B, in, (int)Ly.I, Ly.buf[LANE_BUF_DELTAS], (int)Ly.O,
                     Epi::STORE, Ly.buf[LANE_BUF_G], nullptr, nullptr, nullptr, &mx);
            }
            colsum(g, Ly.buf[LANE_BUF_DELTAS], B, (int)Ly.O, Ly.buf[LANE_BUF_BIAS_GRAD]);
            continue;
        }
        // wgrad sums: G_l = X_l^T D_l ; gb_l = colsum(D_l)
        const GemmMax mx = wgrad_mx(l);
        gemm(g, GemmOp::TN, (int)Ly.I, (int)Ly.O, B, in, (int)Ly.I, Ly.buf[LANE_BUF_DELTAS], (int)Ly.O, Epi::STORE,
             Ly.buf[LANE_BUF_G], nullptr, nullptr, nullptr, &mx);
        colsum(g, Ly.buf[LANE_BUF_DELTAS], B, (int)Ly.O, Ly.buf[LANE_BUF_BIAS_GRAD]);
        if (allreduce) {
            // layer l's G and bias pieces: one contiguous span of the grads arena
            float* begin = Ly.buf[LANE_BUF_G];
            float* end = l + 1 < nl ? net.L(l + 1).buf[LANE_BUF_G] : net.grads + net.grads_count;
            LANE_CUDA(cudaEventRecord(M.ev[l], st));
            LANE_CUDA(cudaStreamWaitEvent(M.comm_stream, M.ev[l], 0));
            LANE_NCCL(ncclAllReduce(begin, begin, static_cast<size_t>(end - begin), ncclFloat32, ncclSum,
                                    c.comm.comm, M.comm_stream));
        }
        if (l > 0) dgrad(l);
    }
    if (allreduce) {
        LANE_CUDA(cudaEventRecord(M.ev[nl], M.comm_stream));
        LANE_CUDA(cudaStreamWaitEvent(st, M.ev[nl], 0));
    }
    c.check_launch();
}

// The update over the whole parameter set in one pass: G = gsum / B_global;
// DW = mu*DW + (-eta)*G (DW = (-eta)*G when mu == 0); W += DW; biases alike.
// With `fused`, only the pieces the wgrad epilogues did not update: every
// bias, and the weights of the layers whose wgrad ran unfused.
template <class Ctx, class Net>
void minibatch_update(Ctx& c, Net& net, size_t B_global, float eta, float mu, const FusedUpdate* fused = nullptr) {
    const float invB = 1.0f / static_cast<float>(B_global);
    // params | grads | velocities are three equal-layout regions (abi.cu arena)
    float* W = net.params;
    float* G = net.grads;
    float* V = net.grads + net.grads_count;
    const size_t n4 = net.params_count / 4;
    const unsigned blocks_max = 4u * static_cast<unsigned>(c.sm_count);
    UpdSpans sp, ps;  // spans to update from gradient sums / from pre-scaled means
    unsigned long long total = 0, ptotal = 0;
    const int nl = static_cast<int>(net.layers.size());
    const bool spans = fused != nullptr;
    auto add = [&](UpdSpans& u, unsigned long long& t, const float* from, const float* to) {
        u.beg[u.n] = static_cast<unsigned long long>(from - W) / 4;
        u.end[u.n] = static_cast<unsigned long long>(to - W) / 4;
        t += u.end[u.n] - u.beg[u.n];
        ++u.n;
    };
    if (spans) {
        for (int l = 0; l < nl; ++l) {
            auto& Ly = net.L(l);
            // [W_l | b_l] or [b_l] alone; pieces are 256-byte aligned, so the
            // end of layer l is the start of layer l+1 (or of the grads region)
            const float* to = l + 1 < nl ? net.L(l + 1).buf[LANE_BUF_W] : net.params + net.params_count;
            if (fused->fused_w[l]) {
                add(sp, total, Ly.buf[LANE_BUF_B], to);
            } else if (fused->scaled_g[l]) {
                add(ps, ptotal, Ly.buf[LANE_BUF_W], Ly.buf[LANE_BUF_B]);
                add(sp, total, Ly.buf[LANE_BUF_B], to);
            } else {
                add(sp, total, Ly.buf[LANE_BUF_W], to);
            }
        }
    }
    if (spans) {
        auto blocks = [&](unsigned long long t) {
            return static_cast<unsigned>(
                std::max<unsigned long long>(1, std::min<unsigned long long>(blocks_max, (t + 255) / 256)));
        };
        k_momentum_update_spans<false><<<blocks(total), 256, 0, c.stream>>>(
            reinterpret_cast<float4*>(W), reinterpret_cast<float4*>(V), reinterpret_cast<float4*>(G), sp, total, invB,
            -eta, mu);
        if (ps.n) {
            k_momentum_update_spans<true><<<blocks(ptotal), 256, 0, c.stream>>>(
                reinterpret_cast<float4*>(W), reinterpret_cast<float4*>(V), reinterpret_cast<float4*>(G), ps, ptotal,
                invB, -eta, mu);
            c.launches += 1;
        }
    } else {
        k_momentum_update_all<<<std::max<size_t>(1, std::min<size_t>(blocks_max, (n4 + 255) / 256)), 256, 0,
                                c.stream>>>(reinterpret_cast<float4*>(W), reinterpret_cast<float4*>(V),
                                            reinterpret_cast<float4*>(G), n4, invB, -eta, mu);
    }
    c.launches += 1;
    c.check_launch();
}

// The whole step on the staged batch.  One rank: the wgrad epilogues apply
// the update of the weights they produce (tensor-core shapes), one small
// kernel the rest.  Data parallel: every layer's gradient span is
// all-reduced (one NCCL allreduce per layer, overlapping the rest of the
// backward), then every rank applies the identical update with
// B_global = B * world.  (LANE_B200_MB_BUCKETS=1 forces the allreduce path on
// a one-rank communicator, where NCCL's sum is the identity.)
// NVLS-bound network (nvls.cuh): barrier (every rank's gradient sums are
// written), this rank's slice of the fused switch-reduce + update + multicast
// store, barrier (every rank's stores have landed before the next forward).
template <class Ctx, class Net>
void minibatch_update_nvls(Ctx& c, Net& net, size_t B_global, float eta, float mu) {
    NvlsState& S = net.nvls;
    const size_t off_flag = net.arena_bytes;  // the counter after the arena
    unsigned* uc_flag = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(S.uc) + off_flag);
    unsigned* mc_flag = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(S.mcva) + off_flag);
    auto mc = [&](const float* p) {
        return reinterpret_cast<float*>(reinterpret_cast<char*>(S.mcva) +
                                        (reinterpret_cast<const char*>(p) - reinterpret_cast<char*>(S.uc)));
    };
    float* W = net.params;
    float* G = net.grads;
    float* V = net.grads + net.grads_count;
    const unsigned long long n4 = net.params_count / 4;
    const unsigned long long beg = n4 * (unsigned long long)S.rank / (unsigned long long)S.world;
    const unsigned long long end = n4 * (unsigned long long)(S.rank + 1) / (unsigned long long)S.world;
    const unsigned blocks = static_cast<unsigned>(std::max<unsigned long long>(
        1, std::min<unsigned long long>(4ull * (unsigned long long)c.sm_count, (end - beg + 255) / 256)));
    const float invB = 1.0f / static_cast<float>(B_global);
    if (!S.local) {
        k_nvls_barrier<true><<<1, 32, 0, c.stream>>>(mc_flag, uc_flag, S.expect, S.world, c.error_flag);
        k_nvls_update<true><<<blocks, 256, 0, c.stream>>>(mc(W), mc(G), mc(V), reinterpret_cast<const float4*>(W),
                                                          reinterpret_cast<const float4*>(V), beg, end, invB, -eta,
                                                          mu);
        k_nvls_barrier<true><<<1, 32, 0, c.stream>>>(mc_flag, uc_flag, S.expect, S.world, c.error_flag);
    } else {
        k_nvls_barrier<false><<<1, 32, 0, c.stream>>>(mc_flag, uc_flag, S.expect, S.world, c.error_flag);
        k_nvls_update<false><<<blocks, 256, 0, c.stream>>>(mc(W), mc(G), mc(V), reinterpret_cast<const float4*>(W),
                                                           reinterpret_cast<const float4*>(V), beg, end, invB, -eta,
                                                           mu);
        k_nvls_barrier<false><<<1, 32, 0, c.stream>>>(mc_flag, uc_flag, S.expect, S.world, c.error_flag);
    }
    c.launches += 3;
    c.check_launch();
}

template <class Ctx, class Net>
void minibatch_body(Ctx& c, Net& net, size_t Bsz, float eta, float mu, double* loss_sum) {
    if (net.nvls.bound) {
        minibatch_grads_body(c, net, Bsz, loss_sum, false);
        minibatch_update_nvls(c, net, Bsz * static_cast<size_t>(net.nvls.world), eta, mu);
        return;
    }
    static const bool force_buckets = std::getenv("LANE_B200_MB_BUCKETS") != nullptr;
    const bool allreduce = c.comm.comm && (c.comm.world > 1 || force_buckets);
    const size_t B_global = Bsz * static_cast<size_t>(c.comm.world);
    if (allreduce || net.layers.size() > static_cast<size_t>(kMaxUpdSpans)) {
        minibatch_grads_body(c, net, Bsz, loss_sum, allreduce);
        minibatch_update(c, net, B_global, eta, mu);
        return;
    }
    FusedUpdate f{1.0f / static_cast<float>(B_global), eta, mu, {}};
    minibatch_grads_body(c, net, Bsz, loss_sum, false, &f);
    minibatch_update(c, net, B_global, eta, mu, &f);
}

}  // namespace lane_b200
