// abi.cu -- implementation of include/lane_b200.h (the C ABI).
//
// One translation unit: the kernels are header-only (.cuh) and instantiated
// here.  Every entry point is wrapped by guard(): C++ exceptions never cross
// the ABI; they become status codes + lane_b200_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "layer_kernels.cuh"
#include "minibatch.cuh"
#include "nvls.cuh"
#include "pipeline.cuh"
#include "sgd_persistent.cuh"
#include "sgd_tiny.cuh"
#include "sgd_window.cuh"

using namespace lane_b200;

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        return LANE_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return LANE_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LANE_ERR_INTERNAL;
    }
}

// ---- host SplitMix64, bit-identical to lane::SeededRng (tensor.hpp:13-44) ----
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t s) : state(s) {}
    uint64_t next_u64() {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    float next_float() { return static_cast<float>(next_u64() >> 40) * 0x1p-24f; }
    // tensor.cpp:7-15 (host float arithmetic; this TU's host code is compiled
    // for baseline x86-64 with -ffp-contract=off: no FMA, like the reference)
    float uniform(float lo, float hi) {
        const float scale = hi - lo;
        const float prod = next_float() * scale;
        const float v = lo + prod;
        return v < hi ? v : std::nextafter(hi, lo);
    }
    size_t below(size_t n) {
        return static_cast<size_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
    }
};

uint64_t fnv1a64(const void* data, size_t len, uint64_t h) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

int blocks_for(size_t n, int threads, int cap) {
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>(cap, (n + threads - 1) / threads)));
}

// G = d (x) x, DW = -eta G (the softmax/fc backward tuples' outer product)
void launch_outer(cudaStream_t st, int sm_count, const float* d, const float* x, float* G, float* DW,
                  float neg_eta, int I, int O) {
    const bool vec = (O & 3) == 0 && ((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(G) |
                                       reinterpret_cast<uintptr_t>(DW)) & 15) == 0;
    if (vec) {
        const int Q = O / 4;
        const unsigned gx = static_cast<unsigned>((Q + 255) / 256);
        const unsigned gy = static_cast<unsigned>(std::min<long long>(
            I, std::max<long long>(1, (long long)16 * sm_count / std::max(1u, gx))));
        k_outer4<<<dim3(gx, std::max(1u, gy)), 256, 0, st>>>(
            reinterpret_cast<const float4*>(d), x, reinterpret_cast<float4*>(G), reinterpret_cast<float4*>(DW),
            neg_eta, I, Q);
    } else {
        k_outer<<<blocks_for(static_cast<size_t>(I) * O, 256, 8 * sm_count), 256, 0, st>>>(d, x, G, DW, neg_eta,
                                                                                           I, O);
    }
}

}  // namespace

#include "dataset.cuh"

// ============================================================== objects ===

struct lane_b200_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int numerics = LANE_NUMERICS_FAST;
    uint64_t launches = 0;
    int sm_count = 148;
    size_t max_smem_optin = 0;
    int* error_flag = nullptr;  // device: set by kernels that bail out
    std::vector<void*> scratch;
    MinibatchComm comm;  // NCCL communicator (mini-batch DP), see minibatch.cuh
    // Networks keep their context alive: ctx_destroy with live networks only
    // marks the context; the last net_destroy releases it (no dangling ctx).
    int live_nets = 0;
    bool destroy_requested = false;

    void count(int n = 1) { launches += static_cast<uint64_t>(n); }
    void check_launch() {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            throw Error(LANE_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    }
    void check_device_error() {
        int flag = 0;
        LANE_CUDA(cudaMemcpyAsync(&flag, error_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
        LANE_CUDA(cudaStreamSynchronize(stream));
        if (flag) {
            LANE_CUDA(cudaMemsetAsync(error_flag, 0, sizeof(int), stream));
            throw Error(LANE_ERR_CUDA, "device exchange timed out (persistent kernel aborted)");
        }
    }
};

// The captured mini-batch step graph and the configuration it was captured for.
struct MbGraph {
    struct Key {
        size_t B = 0;
        float eta = 0, mu = 0;
        double* loss = nullptr;
        int world = 0, numerics = 0, tc = 0;
        const void* comm = nullptr;
        const float* ws = nullptr;  // the GEMM workspace the graph's kernels write
        uint64_t ws_gen = 0;        // and its reallocation count (a freed and reused address)
        bool operator==(const Key& o) const {
            return B == o.B && eta == o.eta && mu == o.mu && loss == o.loss && world == o.world &&
                   numerics == o.numerics && tc == o.tc && comm == o.comm && ws == o.ws && ws_gen == o.ws_gen;
        }
    } key;
    bool warm = false;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        warm = false;
    }
};

struct LayerBufs {
    size_t I = 0, O = 0;
    float* buf[LANE_BUF_COUNT] = {};
    size_t cnt[LANE_BUF_COUNT] = {};
};

struct lane_b200_net {
    lane_b200_ctx* ctx = nullptr;
    size_t input_width = 0, n_hidden = 0, classes = 0, max_batch = 1;
    std::vector<LayerBufs> layers;
    char* arena = nullptr;
    size_t arena_bytes = 0;
    float* params = nullptr;  // [W_0 | b_0 | W_1 | b_1 | ...]
    size_t params_count = 0;
    float* grads = nullptr;  // [G_0 | gb_0 | G_1 | gb_1 | ...] (allreduce target)
    size_t grads_count = 0;
    float* target_stage = nullptr;  // classes * max_batch
    float* scratch = nullptr;       // split-K partials / uploaded next-layer tensors
    size_t scratch_count = 0;
    long long* step = nullptr;
    double* loss_dev = nullptr;
    unsigned long long* correct_dev = nullptr;
    unsigned long long* slots = nullptr;
    size_t slots_count = 0;
    // windowed online-SGD scratch (sgd_window.cuh): banded Gram, Y/d0 rings, counters
    float* win_coef = nullptr;
    size_t win_coef_count = 0;
    float* win_ring = nullptr;
    size_t win_ring_count = 0;
    // dataset staging for train()/evaluate() (uploaded once per call)
    float* data = nullptr;
    size_t data_count = 0;
    uint32_t* order = nullptr;
    size_t order_count = 0;
    MinibatchState mb;  // activations + workspaces of the mini-batch path
    NvlsState nvls;     // NVLS-bound arena (data parallel over NVSwitch multicast)
    MbGraph mb_graph;   // captured mini-batch step (per configuration)
    InputPipeline pipe;  // pinned staging + copy stream of train_minibatch
    std::vector<cudaEvent_t> plan_events;  // backward_plan_run_timed
    float* eval_buf = nullptr;             // batched evaluate scratch
    size_t eval_count = 0;
    float* eval_ws = nullptr;              // batched evaluate GEMM workspace
    size_t eval_ws_count = 0;
    int* eval_counters = nullptr;          // its stream-K tile counters
    size_t eval_counters_count = 0;
    // train(): speculative epochs of small sets (see lane_b200_train)
    float* spec_dev = nullptr;             // K epochs of gathered rows
    size_t spec_dev_count = 0;
    float* spec_host = nullptr;            // page-locked staging of the same
    size_t spec_host_count = 0;
    float* spec_stats = nullptr;           // K x {loss sum, hit count}
    size_t spec_stats_count = 0;
    float* spec_snap = nullptr;            // K arena snapshots (state after each epoch)
    size_t spec_snap_count = 0;

    LayerBufs& L(size_t l) { return layers.at(l); }
    size_t out_layer() const { return n_hidden; }
};

namespace {

void* dev_alloc(size_t bytes) {
    void* p = nullptr;
    LANE_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    return p;
}

void ensure(float*& p, size_t& have, size_t need) {
    if (have >= need) return;
    if (p) LANE_CUDA(cudaFree(p));
    p = static_cast<float*>(dev_alloc(need * sizeof(float)));
    have = need;
}

void check_eta(float eta) {
    // LearningRate (layers.hpp:11-19)
    if (!(eta > 0.0f)) throw Error(LANE_ERR_CONFIG, "LearningRate: eta must be positive");
}

void check_mu(float mu) {
    // momentum (extension): finite, 0 <= mu < 1 (NaN fails too)
    if (!(mu >= 0.0f && mu < 1.0f)) throw Error(LANE_ERR_CONFIG, "momentum: mu must be in [0, 1)");
}

void check_layer(lane_b200_net* net, size_t layer) {
    if (!net) throw Error(LANE_ERR_CONFIG, "null network");
    if (layer >= net->layers.size()) throw Error(LANE_ERR_CONFIG, "layer index out of range");
}

// ---------------------------------------------------------------- layers ---

void run_layer_forward(lane_b200_net* net, size_t l, const float* src) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& Ly = net->L(l);
    const int I = static_cast<int>(Ly.I), O = static_cast<int>(Ly.O);
    const bool softmax = l == net->out_layer();
    const int act = softmax ? ACT_NONE : ACT_TANH;
    const bool strict = c->numerics == LANE_NUMERICS_STRICT;
    float* z = Ly.buf[LANE_BUF_NETIN];
    float* a = Ly.buf[LANE_BUF_OUTPUTS];
    if (strict || I < 512) {
        // thread per output, sequential i: exact reference order (and the
        // fastest choice when I is small)
        k_netin_strict<<<blocks_for(O, 128, 1 << 20), 128, 0, c->stream>>>(
            src, Ly.buf[LANE_BUF_INPUTS], Ly.buf[LANE_BUF_W], Ly.buf[LANE_BUF_B], z, a, I, O, act);
        c->count();
    } else {
        const int colblocks = (O + 31) / 32;
        int S = std::max(1, std::min((2 * c->sm_count + colblocks - 1) / colblocks, I / 64));
        const int chunk = (I + S - 1) / S;
        S = (I + chunk - 1) / chunk;
        ensure(net->scratch, net->scratch_count, static_cast<size_t>(S) * O);
        k_netin_fast_part<<<dim3(colblocks, S), dim3(32, 8), 0, c->stream>>>(src, Ly.buf[LANE_BUF_W],
                                                                            net->scratch, I, O, chunk);
        k_netin_fast_finish<<<blocks_for(O, 128, 1 << 20), 128, 0, c->stream>>>(
            net->scratch, S, src, Ly.buf[LANE_BUF_INPUTS], I, Ly.buf[LANE_BUF_B], z, a, O, act);
        c->count(2);
    }
    if (softmax) {
        const int th = std::min(1024, ((O + 31) / 32) * 32);
        k_softmax<<<1, th, 0, c->stream>>>(z, a, O, strict ? 1 : 0);
        c->count();
    }
    c->check_launch();
}

void run_fc_backward(lane_b200_net* net, size_t l, const float* nW, const float* nd, int N,
                     float eta) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& Ly = net->L(l);
    const int I = static_cast<int>(Ly.I), O = static_cast<int>(Ly.O);
    const float neg_eta = -eta;
    if (c->numerics == LANE_NUMERICS_STRICT || N < 64) {
        k_delta_fc_strict<<<blocks_for(O, 128, 1 << 20), 128, 0, c->stream>>>(
            Ly.buf[LANE_BUF_OUTPUTS], nW, nd, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_DELTA_BIASES],
            neg_eta, O, N);
    } else {
        k_delta_fc_fast<<<blocks_for(static_cast<size_t>(O) * 32, 256, 1 << 20), 256, 0, c->stream>>>(
            Ly.buf[LANE_BUF_OUTPUTS], nW, nd, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_DELTA_BIASES],
            neg_eta, O, N);
    }
    launch_outer(c->stream, c->sm_count, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_INPUTS], Ly.buf[LANE_BUF_G],
                 Ly.buf[LANE_BUF_DW], neg_eta, I, O);
    c->count(2);
    c->check_launch();
}

void run_softmax_backward(lane_b200_net* net, const float* t_dev, float eta) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& Ly = net->L(net->out_layer());
    const int I = static_cast<int>(Ly.I), O = static_cast<int>(Ly.O);
    k_delta_softmax<<<blocks_for(O, 128, 1 << 20), 128, 0, c->stream>>>(
        Ly.buf[LANE_BUF_OUTPUTS], t_dev, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_DELTA_BIASES], -eta, O);
    launch_outer(c->stream, c->sm_count, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_INPUTS], Ly.buf[LANE_BUF_G],
                 Ly.buf[LANE_BUF_DW], -eta, I, O);
    c->count(2);
    c->check_launch();
}

void run_apply_updates(lane_b200_net* net, size_t l) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& Ly = net->L(l);
    const size_t n = Ly.I * Ly.O;
    k_apply_updates<<<blocks_for(n / 4 + Ly.O, 256, 8 * c->sm_count), 256, 0, c->stream>>>(
        Ly.buf[LANE_BUF_W], Ly.buf[LANE_BUF_DW], n, Ly.buf[LANE_BUF_B], Ly.buf[LANE_BUF_DELTA_BIASES],
        static_cast<int>(Ly.O));
    c->count();
    c->check_launch();
}

void run_backward_plan(lane_b200_net* net, const float* t_dev, float eta) {
    // BackwardPlan::run (network.cpp:122-138)
    run_softmax_backward(net, t_dev, eta);
    for (size_t l = net->n_hidden; l-- > 0;) {
        LayerBufs& nx = net->L(l + 1);
        run_fc_backward(net, l, nx.buf[LANE_BUF_W], nx.buf[LANE_BUF_DELTAS], static_cast<int>(nx.O), eta);
    }
    for (size_t l = 0; l < net->layers.size(); ++l) run_apply_updates(net, l);
}

void run_forward_chain(lane_b200_net* net) {
    for (size_t l = 0; l < net->layers.size(); ++l) {
        const float* src = l == 0 ? net->L(0).buf[LANE_BUF_INPUTS] : net->L(l - 1).buf[LANE_BUF_OUTPUTS];
        run_layer_forward(net, l, src);
    }
}

// ------------------------------------------------ fused persistent path ---

struct SgdPlan {
    bool ok = false;
    bool window = false;   // delayed-base windowed kernel (chain CTA + W0 producers)
    int jpl = 4, D = 3;    // window plan: hidden units per chain lane, lag in blocks
    int ncw = 1;           // window plan: chain warps
    int cs = 1, qpc = 1;   // window plan: chain CTAs (cluster), column quads per producer
    int ks = 1, rpc = 0;   // window plan: producer row splits per column quad, rows per split
    bool cluster = false;  // single thread-block cluster, DSMEM exchange
    bool w0_smem = true;   // grid plan: W0 slices resident in shared memory
    bool col4 = false;     // grid streamed plan: 128-bit column quads
    int chunks = 1;        // grid streamed plan: K chunks per column group
    int G = 0, npc = 0, wpn = 1;
    size_t smem = 0;
};

int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

using SgdKernel = void (*)(SgdArgs);

SgdKernel cluster_kernel(int C) {
    // the reference's benchmark topologies are 10-class; other class counts
    // use the runtime-C instantiation
    return C == 10 ? k_sgd_cluster<10> : C == 3 ? k_sgd_cluster<3> : k_sgd_cluster<0>;
}

// Sets the kernel's opt-in attributes (every call: the attributes are
// per-device function state) and reports whether one cluster of CS CTAs with
// `smem` bytes fits.  The occupancy answer is cached per (device, kernel, CS,
// smem) under a mutex.
bool cluster_fits(SgdKernel kern, int CS, size_t smem) {
    LANE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    LANE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    int dev = 0;
    LANE_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<std::tuple<int, SgdKernel, int, size_t>, bool> cache;
    const auto key = std::make_tuple(dev, kern, CS, smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    cudaGetLastError();
    const bool ok = e == cudaSuccess && n >= 1;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = ok;
    return ok;
}

SgdKernel grid_kernel(int C, bool w0_smem) {
    if (w0_smem) return C == 10 ? k_sgd_grid<10, true> : k_sgd_grid<0, true>;
    return C == 10 ? k_sgd_grid<10, false> : k_sgd_grid<0, false>;
}

using WinKernel = void (*)(WinArgs);
constexpr int kWinWideQPC = 8;  // wide producers: 8 column quads x 2 W0 rows per thread

// co-resident CTAs of a cluster launch of the windowed kernel (cluster size cs)
int window_cluster_capacity(int cs, size_t smem) {
    const WinKernel kern = k_sgd_window<4, 10, 1, true, kWinMaxQPC>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int dev = 0;
    LANE_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<std::tuple<int, int, size_t>, int> cache;  // (device, cs, smem) -> CTAs
    const auto key = std::make_tuple(dev, cs, smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(win_threads<1>());
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess) nclusters = 0;
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = nclusters * cs;
    return nclusters * cs;
}

SgdPlan plan_persistent(lane_b200_net* net) {
    SgdPlan p;
    lane_b200_ctx* c = net->ctx;
    if (net->n_hidden != 1 || c->numerics != LANE_NUMERICS_FAST) return p;
    const int I = static_cast<int>(net->input_width), H = static_cast<int>(net->L(0).O),
              C = static_cast<int>(net->classes);
    if (C > kClMaxC) return p;
    const char* mode = std::getenv("LANE_B200_SGD_MODE");
    if (!mode || std::strcmp(mode, "window") == 0) {
        // windowed plan: the chain on one CTA, W0 on H/4 producer CTAs
        // window depth D: 2 measured best at C2 and up to 1024 units (producers
        // keep up with one block of lag); the 16-CTA cluster chains (H >= 2048)
        // run 9-15% faster with D = 3 (more lag for the producers' pass), when
        // the deeper rings fit in shared memory (not at H = 8192)
        const char* env_d = std::getenv("LANE_B200_SGD_WIN_D");
        const bool wide = H > 256 && next_pow2((H + 127) / 128) >= kWinMaxCS;
        const int nD = wide && !env_d ? 2 : 1;  // D = 3, then 2; or just 2 (or the override)
        for (int di = 0; di < nD; ++di) {
            const int D = env_d ? std::max(2, std::min(std::atoi(env_d), kWinMaxD)) : (nD == 2 && di == 0 ? 3 : 2);
            // chain geometry: H <= 128 -> one chain warp x 4 units/lane; <= 256 ->
            // two warps x 4 (measured at C2: one warp 1.83M samples/s, two 1.68M --
            // the barrier and the duplicated softmax outweigh the halved H work);
            // wider -> CS = H/128 chain CTAs in one cluster, one warp each, with a
            // DSMEM exchange of the slice partial logits per sample
            int cs = 1;
            if (H > 256) cs = std::min(kWinMaxCS, next_pow2((H + 127) / 128));
            const int Hs = H / cs;
            // one chain warp per 128 units of a cluster slice (1, 2 or 4)
            int ncw = cs > 1 ? (Hs <= 128 ? 1 : Hs <= 256 ? 2 : Hs <= 512 ? 4 : 8) : (H <= 128 ? 1 : 2);
            if (const char* e = std::getenv("LANE_B200_SGD_WIN_NCW"))
                if (cs == 1) ncw = (std::atoi(e) == 1 && H <= 128) ? 1 : 2;
            const int jpl = ncw == 1 ? 4 : ((cs == 1 && H <= 128) ? 2 : 4);
            // producers: H/4 column quads (QPC per CTA) x KS row splits (<= 2
            // splits, >= 32 rows each); rows per split a multiple of 4 (cp.async 16 B)
            const int quads = std::max(1, H / 4);
            int pmax = c->sm_count - cs;
            int ks = std::max(1, std::min({2, pmax / quads, std::max(1, I / 32)}));
            if (const char* e = std::getenv("LANE_B200_SGD_WIN_KS")) ks = std::max(1, std::min(std::atoi(e), 2));
            const int rpc = (((I + ks - 1) / ks) + 3) & ~3;
            ks = (I + rpc - 1) / rpc;
            // (the d0-direct choice needs the producer variant: wide/smem producers
            // when the quads per producer exceed 4 -- known after the capacity query;
            // size the chain CTA for the non-direct ring, the larger of the two)
            const WinSmem L(32 * jpl * ncw, D, ks, Hs, ncw, cs > 1 && ncw >= 2);
            const size_t psmem_reg = ProdSmem(rpc, D).total;
            // producers: register slices up to kWinWideQPC quads, else W0 in smem
            // (the quad count is only known after the capacity query; size for both)
            const size_t smem_reg = std::max(L.total, psmem_reg);
            // co-resident CTAs: one per SM; clusters of cs must also fit the GPCs
            int max_ctas = c->sm_count;
            if (cs > 1 && cs <= kWinMaxCS && smem_reg <= c->max_smem_optin)
                max_ctas = std::min(max_ctas, window_cluster_capacity(cs, smem_reg));
            pmax = std::max(1, max_ctas - cs);
            const int qpc = std::max(1, (quads * ks + pmax - 1) / pmax);
            const int producers = ((quads + qpc - 1) / qpc) * ks;
            const int grid = ((cs + producers + cs - 1) / cs) * cs;  // a whole number of clusters
            const bool psm = qpc > kWinWideQPC;  // W0 slices in shared memory
            const size_t smem = psm ? std::max(L.total, ProdSmemS(rpc, D, qpc).total) : smem_reg;
            const int nthr = ncw == 4 ? 320 : ncw == 2 ? 256 : 224;
            if (ncw <= 4 && H % (4 * cs) == 0 && Hs <= 32 * jpl * ncw && cs <= kWinMaxCS && C <= kWinCP &&
                rpc <= (qpc > kWinMaxQPC ? 2 : kWinMaxNR) * nthr &&
                qpc <= (cs > 1 ? kWinSmemQPC : 1) && (cs == 1 || ncw == 1 || psm) &&
                grid <= max_ctas && smem <= c->max_smem_optin) {
                p.ok = p.window = true;
                p.jpl = jpl;
                p.ncw = ncw;
                p.cs = cs;
                p.qpc = qpc;
                p.D = D;
                p.ks = ks;
                p.rpc = rpc;
                p.G = grid;
                p.smem = smem;
                return p;
            }
        }
        if (mode) return p;
    }
    if (!mode || std::strcmp(mode, "cluster") == 0) {
        // single-cluster plan: the whole hidden layer on <= 16 SMs, DSMEM exchange
        int CS = std::min(16, H);
        if (const char* e = std::getenv("LANE_B200_SGD_CLUSTER")) CS = std::max(1, std::min(std::atoi(e), std::min(16, H)));
        const int npc = (H + CS - 1) / CS;
        CS = (H + npc - 1) / npc;
        const int wpn = npc >= kClBulkWarps ? 1 : kClBulkWarps / next_pow2(npc);
        const ClSmem L(I, C, npc, wpn, CS);
        if (L.total <= c->max_smem_optin && cluster_fits(cluster_kernel(C), CS, L.total)) {
            p.ok = p.cluster = true;
            p.G = CS;
            p.npc = npc;
            p.wpn = wpn;
            p.smem = L.total;
            return p;
        }
        if (mode) return p;
    }
    // grid plan: every SM, L2 exchange; W0 in shared memory when it fits,
    // otherwise streamed from HBM each sample
    int G = std::min(c->sm_count, H);
    if (const char* e = std::getenv("LANE_B200_SGD_CTAS")) G = std::max(1, std::min(std::atoi(e), std::min(c->sm_count, H)));
    int npc = (H + G - 1) / G;
    if (H % 4 == 0) npc = (npc + 3) & ~3;  // 128-bit column quads in the streamed pass
    G = (H + npc - 1) / npc;
    // streamed pass: enough (column group, K chunk) items for ~2 rounds of
    // the 512 bulk threads, as far as shared memory allows
    p.col4 = H % 4 == 0;
    const int groups = p.col4 ? npc / 4 : npc;
    int chunks = std::max(1, std::min(kGrChunks, (2 * 32 * kClBulkWarps + groups / 2) / std::max(1, groups)));
    chunks = std::min(chunks, std::max(1, I / 8));
    while (chunks > 1 && GrSmem(I, C, npc, G, false, chunks).total > c->max_smem_optin) --chunks;
    const GrSmem Ls(I, C, npc, G, true), Lg(I, C, npc, G, false, chunks);
    const bool force_stream = std::getenv("LANE_B200_SGD_STREAM") != nullptr;
    if (!force_stream && Ls.total <= c->max_smem_optin) {
        p.w0_smem = true;
        p.smem = Ls.total;
        p.chunks = 1;
    } else if (Lg.total <= c->max_smem_optin) {
        p.w0_smem = false;
        p.smem = Lg.total;
        p.chunks = chunks;
    } else {
        return p;
    }
    p.ok = true;
    p.G = G;
    p.npc = npc;
    return p;
}

void launch_persistent(lane_b200_net* net, const SgdPlan& P, const float* X, const float* T, size_t n,
                       const uint32_t* order, size_t n_steps, float eta, double* loss_sum,
                       unsigned long long* correct) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& L0 = net->L(0);
    LayerBufs& L1 = net->L(1);
    const size_t need = 2ull * P.G * net->classes;
    if (net->slots_count < need) {
        if (net->slots) LANE_CUDA(cudaFree(net->slots));
        net->slots = static_cast<unsigned long long*>(dev_alloc(need * 8));
        net->slots_count = need;
    }
    LANE_CUDA(cudaMemsetAsync(net->slots, 0, need * 8, c->stream));
    SgdArgs A{};
    A.I = static_cast<int>(net->input_width);
    A.H = static_cast<int>(L0.O);
    A.C = static_cast<int>(net->classes);
    A.G = P.G;
    A.npc = P.npc;
    A.wpn = P.wpn;
    A.X = X;
    A.T = T;
    A.order = order;
    A.n = static_cast<long long>(n);
    A.n_steps = static_cast<long long>(n_steps);
    A.neg_eta = -eta;
    A.W0 = L0.buf[LANE_BUF_W];
    A.b0 = L0.buf[LANE_BUF_B];
    A.W1 = L1.buf[LANE_BUF_W];
    A.b1 = L1.buf[LANE_BUF_B];
    A.slots = net->slots;
    A.x0 = L0.buf[LANE_BUF_INPUTS];
    A.z0 = L0.buf[LANE_BUF_NETIN];
    A.a0 = L0.buf[LANE_BUF_OUTPUTS];
    A.d0 = L0.buf[LANE_BUF_DELTAS];
    A.db0 = L0.buf[LANE_BUF_DELTA_BIASES];
    A.x1 = L1.buf[LANE_BUF_INPUTS];
    A.z1 = L1.buf[LANE_BUF_NETIN];
    A.a1 = L1.buf[LANE_BUF_OUTPUTS];
    A.d1 = L1.buf[LANE_BUF_DELTAS];
    A.db1 = L1.buf[LANE_BUF_DELTA_BIASES];
    A.loss_sum = loss_sum;
    A.correct = correct;
    A.error = c->error_flag;
    const char* trace_path = std::getenv("LANE_B200_SGD_TRACE");
    unsigned long long* trace = nullptr;
    const size_t trace_n = static_cast<size_t>(kTraceSamples) * kTracePhases;
    if (trace_path) {
        trace = static_cast<unsigned long long*>(dev_alloc(trace_n * 8));
        LANE_CUDA(cudaMemsetAsync(trace, 0, trace_n * 8, c->stream));
    }
    A.trace = trace;
    A.chunks = P.chunks;
    A.debug = std::getenv("LANE_B200_SGD_DEBUG") ? std::atoi(std::getenv("LANE_B200_SGD_DEBUG")) : 0;
    A.col4 = P.col4 ? 1 : 0;
    if (P.cluster) {
        const SgdKernel kern = cluster_kernel(A.C);
        cluster_fits(kern, P.G, P.smem);  // sets the function attributes
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(P.G);
        cfg.blockDim = dim3(kClThreads);
        cfg.dynamicSmemBytes = P.smem;
        cfg.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = P.G;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        LANE_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    } else {
        const SgdKernel kern = grid_kernel(A.C, P.w0_smem);
        LANE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(P.smem)));
        int per_sm = 0;
        LANE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kClThreads, P.smem));
        if (per_sm < 1 || P.G > per_sm * c->sm_count)
            throw Error(LANE_ERR_CUDA, "grid SGD kernel cannot be co-resident");
        void* args[] = {&A};
        LANE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(P.G), dim3(kClThreads), args,
                                              P.smem, c->stream));
    }
    c->count();
    if (trace) {  // debug: per-phase cycle stamps of CTA 0
        std::vector<unsigned long long> h(trace_n);
        LANE_CUDA(cudaMemcpyAsync(h.data(), trace, trace_n * 8, cudaMemcpyDeviceToHost, c->stream));
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        LANE_CUDA(cudaFree(trace));
        if (FILE* f = std::fopen(trace_path, "a")) {
            std::fprintf(f, "# plan cluster=%d G=%d npc=%d wpn=%d\n", P.cluster ? 1 : 0, P.G, P.npc, P.wpn);
            for (int s = 0; s < kTraceSamples; ++s) {
                for (int ph = 0; ph < kTracePhases; ++ph) std::fprintf(f, "%llu ", h[s * kTracePhases + ph]);
                std::fprintf(f, "\n");
            }
            std::fclose(f);
        }
    }
    // G and DW of the last sample, as the reference's stream_out leaves them
    for (size_t l = 0; l < 2; ++l) {
        LayerBufs& Ly = net->L(l);
        launch_outer(c->stream, c->sm_count, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_INPUTS],
                     Ly.buf[LANE_BUF_G], Ly.buf[LANE_BUF_DW], -eta, static_cast<int>(Ly.I), static_cast<int>(Ly.O));
        c->count();
    }
    c->check_launch();
}

// cluster chains: producers with up to 4 quads x 4 rows/thread, or 8 quads x 2 rows
WinKernel window_kernel(int jpl, int ncw, int C, int cs, int qpc) {
    if (cs > 1 && qpc > kWinWideQPC) {
        if (ncw == 4)
            return C == 10 ? k_sgd_window<4, 10, 4, true, kWinSmemQPC, 2> : k_sgd_window<4, 0, 4, true, kWinSmemQPC, 2>;
        if (ncw == 2)
            return C == 10 ? k_sgd_window<4, 10, 2, true, kWinSmemQPC, 2> : k_sgd_window<4, 0, 2, true, kWinSmemQPC, 2>;
        return C == 10 ? k_sgd_window<4, 10, 1, true, kWinSmemQPC, 2> : k_sgd_window<4, 0, 1, true, kWinSmemQPC, 2>;
    }
    if (cs > 1 && qpc > kWinMaxQPC)
        return C == 10 ? k_sgd_window<4, 10, 1, true, kWinWideQPC, 2> : k_sgd_window<4, 0, 1, true, kWinWideQPC, 2>;
    if (cs > 1)
        return C == 10 ? k_sgd_window<4, 10, 1, true, kWinMaxQPC> : k_sgd_window<4, 0, 1, true, kWinMaxQPC>;
    if (ncw == 1) return C == 10 ? k_sgd_window<4, 10, 1> : C == 3 ? k_sgd_window<4, 3, 1> : k_sgd_window<4, 0, 1>;
    if (jpl == 2) return C == 10 ? k_sgd_window<2, 10, 2> : k_sgd_window<2, 0, 2>;
    return C == 10 ? k_sgd_window<4, 10, 2> : k_sgd_window<4, 0, 2>;
}

void launch_window(lane_b200_net* net, const SgdPlan& P, const float* X, const float* T, size_t n,
                   const uint32_t* order, size_t n_steps, long long base, float eta, double* loss_sum,
                   unsigned long long* correct) {
    lane_b200_ctx* c = net->ctx;
    LayerBufs& L0 = net->L(0);
    LayerBufs& L1 = net->L(1);
    const int H = static_cast<int>(L0.O);
    const int QW = P.D * kWinS;
    ensure(net->win_coef, net->win_coef_count, n_steps * QW);
    const size_t yring = static_cast<size_t>(P.D + 1) * P.ks * kWinS * H;  // partial Y per row split
    const size_t dring = static_cast<size_t>(P.D + 1) * kWinS * H;
    const size_t cnt_words = 64;  // ycnt[D+1] | dcnt (32-bit), padded
    ensure(net->win_ring, net->win_ring_count, yring + dring + cnt_words);
    unsigned* cnt = reinterpret_cast<unsigned*>(net->win_ring + yring + dring);
    LANE_CUDA(cudaMemsetAsync(cnt, 0, cnt_words * sizeof(float), c->stream));
    WinArgs A{};
    A.I = static_cast<int>(net->input_width);
    A.H = H;
    A.C = static_cast<int>(net->classes);
    A.D = P.D;
    A.KS = P.ks;
    A.RPC = P.rpc;
    A.QPC = P.qpc;
    A.CS = P.cs;
    A.P = ((H / 4 + P.qpc - 1) / P.qpc) * P.ks;  // active producers
    A.QW = QW;
    A.X = X;
    A.T = T;
    A.order = order;
    if (n >= (size_t(1) << 31) || n_steps > (size_t(1) << 18))
        throw Error(LANE_ERR_CONFIG, "sgd_stream: dataset too large for the windowed kernel");
    A.n = static_cast<int>(n);
    A.n_steps = static_cast<int>(n_steps);
    A.base = static_cast<int>(base);
    A.neg_eta = -eta;
    A.W0 = L0.buf[LANE_BUF_W];
    A.b0 = L0.buf[LANE_BUF_B];
    A.W1 = L1.buf[LANE_BUF_W];
    A.b1 = L1.buf[LANE_BUF_B];
    A.coef = net->win_coef;
    A.yring = net->win_ring;
    A.dring = net->win_ring + yring;
    A.ycnt = cnt;
    A.dcnt = cnt + 32;
    A.x0 = L0.buf[LANE_BUF_INPUTS];
    A.z0 = L0.buf[LANE_BUF_NETIN];
    A.a0 = L0.buf[LANE_BUF_OUTPUTS];
    A.d0 = L0.buf[LANE_BUF_DELTAS];
    A.db0 = L0.buf[LANE_BUF_DELTA_BIASES];
    A.x1 = L1.buf[LANE_BUF_INPUTS];
    A.z1 = L1.buf[LANE_BUF_NETIN];
    A.a1 = L1.buf[LANE_BUF_OUTPUTS];
    A.d1 = L1.buf[LANE_BUF_DELTAS];
    A.db1 = L1.buf[LANE_BUF_DELTA_BIASES];
    A.loss_sum = loss_sum;
    A.correct = correct;
    A.error = c->error_flag;
    const char* trace_path = std::getenv("LANE_B200_SGD_TRACE");
    const size_t trace_n = static_cast<size_t>(kTraceSamples) * kTracePhases;
    if (trace_path) {
        A.trace = static_cast<unsigned long long*>(dev_alloc(trace_n * 8));
        LANE_CUDA(cudaMemsetAsync(A.trace, 0, trace_n * 8, c->stream));
        if (const char* e = std::getenv("LANE_B200_SGD_TRACE_BASE")) A.trace_base = std::atoi(e);
    }
    // banded Gram pre-pass
    {
        const dim3 g(static_cast<unsigned>((n_steps + kGramTS - 1) / kGramTS));
        switch ((QW + 7) / 8) {
            case 2: k_gram_band<2><<<g, 256, 0, c->stream>>>(A); break;
            case 4: k_gram_band<4><<<g, 256, 0, c->stream>>>(A); break;
            case 6: k_gram_band<6><<<g, 256, 0, c->stream>>>(A); break;
            case 8: k_gram_band<8><<<g, 256, 0, c->stream>>>(A); break;
            case 10: k_gram_band<10><<<g, 256, 0, c->stream>>>(A); break;
            case 12: k_gram_band<12><<<g, 256, 0, c->stream>>>(A); break;
            default: throw Error(LANE_ERR_INTERNAL, "window: unsupported Gram band width");
        }
    }
    c->count();
    const WinKernel kern = (A.trace && P.jpl == 4 && P.ncw == 1 && P.cs == 1 && A.C == 10)
                               ? k_sgd_window<4, 10, 1, false, 1, kWinMaxNR, true>
                               : window_kernel(P.jpl, P.ncw, A.C, P.cs, P.qpc);
    LANE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P.smem)));
    void* args[] = {&A};
    const int nthreads = P.ncw == 4 ? win_threads<4>() : P.ncw == 2 ? win_threads<2>() : win_threads<1>();
    if (P.cs == 1) {
        LANE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(P.G), dim3(nthreads), args,
                                              P.smem, c->stream));
    } else {
        // chain CTAs form one cluster (CTAs 0..CS-1); every CTA co-resident
        LANE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(P.G);
        cfg.blockDim = dim3(nthreads);
        cfg.dynamicSmemBytes = P.smem;
        cfg.stream = c->stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = P.cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        LANE_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    }
    c->count();
    if (A.trace) {
        std::vector<unsigned long long> h(trace_n);
        LANE_CUDA(cudaMemcpyAsync(h.data(), A.trace, trace_n * 8, cudaMemcpyDeviceToHost, c->stream));
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        LANE_CUDA(cudaFree(A.trace));
        if (FILE* f = std::fopen(trace_path, "a")) {
            std::fprintf(f, "# plan window G=%d jpl=%d D=%d\n", P.G, P.jpl, P.D);
            for (int s = 0; s < kTraceSamples; ++s) {
                for (int ph = 0; ph < kTracePhases; ++ph) std::fprintf(f, "%llu ", h[s * kTracePhases + ph]);
                std::fprintf(f, "\n");
            }
            std::fclose(f);
        }
    }
    c->check_launch();
}

// G and DW of the last sample, as the reference's stream_out leaves them
void materialise_last_grads(lane_b200_net* net, float eta) {
    lane_b200_ctx* c = net->ctx;
    for (size_t l = 0; l < 2; ++l) {
        LayerBufs& Ly = net->L(l);
        launch_outer(c->stream, c->sm_count, Ly.buf[LANE_BUF_DELTAS], Ly.buf[LANE_BUF_INPUTS],
                     Ly.buf[LANE_BUF_G], Ly.buf[LANE_BUF_DW], -eta, static_cast<int>(Ly.I), static_cast<int>(Ly.O));
        c->count();
    }
    c->check_launch();
}

// Per-sample layer-kernel stream (STRICT numerics, deep nets, C > 128 or
// slices that do not fit on chip): one captured CUDA graph per step.
void stream_layer_path(lane_b200_net* net, const float* X, const float* T, size_t n,
                       const uint32_t* order, size_t n_steps, float eta, double* loss_sum,
                       unsigned long long* correct, bool train) {
    lane_b200_ctx* c = net->ctx;
    LANE_CUDA(cudaMemsetAsync(net->step, 0, sizeof(long long), c->stream));
    const int I = static_cast<int>(net->input_width), C = static_cast<int>(net->classes);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    const uint64_t before = c->launches;
    LANE_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
        k_stage_sample<<<1, 256, 0, c->stream>>>(X, T, order, static_cast<long long>(n), net->step,
                                                 net->L(0).buf[LANE_BUF_INPUTS], I, net->target_stage, C);
        c->count();
        run_forward_chain(net);
        LayerBufs& out = net->L(net->out_layer());
        if (loss_sum || correct) {
            k_loss_accumulate<<<1, 32, 0, c->stream>>>(out.buf[LANE_BUF_OUTPUTS], net->target_stage, C,
                                                       loss_sum, correct);
            c->count();
        }
        if (train) run_backward_plan(net, net->target_stage, eta);
        k_step_advance<<<1, 32, 0, c->stream>>>(net->step);
        c->count();
    } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    LANE_CUDA(cudaStreamEndCapture(c->stream, &graph));
    const uint64_t per_step = c->launches - before;
    c->launches = before;
    LANE_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    for (size_t s = 0; s < n_steps; ++s) LANE_CUDA(cudaGraphLaunch(exec, c->stream));
    c->count(static_cast<int>(per_step * n_steps));
    LANE_CUDA(cudaGraphExecDestroy(exec));
    LANE_CUDA(cudaGraphDestroy(graph));
}

// the one-warp kernel for tiny one-hidden-layer nets in STRICT numerics (it
// computes in the reference's order, bit for bit); LANE_B200_SGD_MODE
// selects another plan
bool tiny_plan(const lane_b200_net* net) {
    if (net->n_hidden != 1 || net->ctx->numerics != LANE_NUMERICS_STRICT) return false;
    const char* mode = std::getenv("LANE_B200_SGD_MODE");
    if (mode && std::strcmp(mode, "tiny") != 0) return false;
    return tiny_fits(static_cast<int>(net->input_width), static_cast<int>(net->layers[0].O),
                     static_cast<int>(net->classes));
}

void sgd_stream_impl(lane_b200_net* net, const float* X, const float* T, size_t n, const uint32_t* order,
                     size_t n_steps, float eta, double* loss_sum, unsigned long long* correct) {
    check_eta(eta);
    if (n == 0) throw Error(LANE_ERR_TRAINING, "sgd_stream: empty sample set");
    if (!X || !T) throw Error(LANE_ERR_CONFIG, "sgd_stream: null data");
    if (n_steps == 0) return;
    if (tiny_plan(net)) {
        // one warp for the whole stream, reference arithmetic (sgd_tiny.cuh)
        lane_b200_ctx* c = net->ctx;
        LayerBufs& L0 = net->L(0);
        LayerBufs& L1 = net->L(1);
        TinyArgs A{};
        A.I = static_cast<int>(net->input_width);
        A.H = static_cast<int>(L0.O);
        A.C = static_cast<int>(net->classes);
        A.X = X;
        A.T = T;
        A.order = order;
        A.n = static_cast<long long>(n);
        A.n_steps = static_cast<long long>(n_steps);
        A.base = 0;
        A.neg_eta = -eta;
        A.W0 = L0.buf[LANE_BUF_W];
        A.b0 = L0.buf[LANE_BUF_B];
        A.W1 = L1.buf[LANE_BUF_W];
        A.b1 = L1.buf[LANE_BUF_B];
        A.x0 = L0.buf[LANE_BUF_INPUTS];
        A.z0 = L0.buf[LANE_BUF_NETIN];
        A.a0 = L0.buf[LANE_BUF_OUTPUTS];
        A.d0 = L0.buf[LANE_BUF_DELTAS];
        A.db0 = L0.buf[LANE_BUF_DELTA_BIASES];
        A.G0 = L0.buf[LANE_BUF_G];
        A.DW0 = L0.buf[LANE_BUF_DW];
        A.x1 = L1.buf[LANE_BUF_INPUTS];
        A.z1 = L1.buf[LANE_BUF_NETIN];
        A.a1 = L1.buf[LANE_BUF_OUTPUTS];
        A.d1 = L1.buf[LANE_BUF_DELTAS];
        A.db1 = L1.buf[LANE_BUF_DELTA_BIASES];
        A.G1 = L1.buf[LANE_BUF_G];
        A.DW1 = L1.buf[LANE_BUF_DW];
        A.loss_sum = loss_sum;
        A.correct = correct;
        tiny_launch(c->stream, A);
        c->count();
        c->check_launch();
        return;
    }
    const SgdPlan P = plan_persistent(net);
    if (P.ok && P.window) {
        // the banded Gram scratch is sized per launch: stream in chunks
        const size_t chunk = size_t(1) << 18;
        for (size_t done = 0; done < n_steps; done += chunk) {
            const size_t m = std::min(chunk, n_steps - done);
            launch_window(net, P, X, T, n, order ? order + done : nullptr, m, static_cast<long long>(done % n),
                          eta, loss_sum, correct);
        }
        materialise_last_grads(net, eta);
    } else if (P.ok) {
        // the persistent kernels index samples with 32-bit counters
        const size_t chunk = size_t(1) << 30;
        for (size_t done = 0; done < n_steps; done += chunk) {
            const size_t m = std::min(chunk, n_steps - done);
            if (order) {
                launch_persistent(net, P, X, T, n, order + done, m, eta, loss_sum, correct);
            } else {
                if (done % n != 0) throw Error(LANE_ERR_CONFIG, "sgd_stream: stream too long for one call");
                launch_persistent(net, P, X, T, n, nullptr, m, eta, loss_sum, correct);
            }
        }
    }
    else
        stream_layer_path(net, X, T, n, order, n_steps, eta, loss_sum, correct, true);
}

}  // namespace

// ============================================================ the ABI ===

extern "C" {

int lane_b200_abi_version(void) { return LANE_B200_ABI_VERSION; }

const char* lane_b200_last_error(void) { return g_last_error.c_str(); }

int lane_b200_ctx_create(int device, lane_b200_ctx** out) {
    return guard([&] {
        if (!out) throw Error(LANE_ERR_CONFIG, "null out");
        int ndev = 0;
        LANE_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw Error(LANE_ERR_CONFIG, "no such CUDA device");
        LANE_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        LANE_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw Error(LANE_ERR_CONFIG, "lane_b200 is built for sm_100a (B200) only");
        auto* c = new lane_b200_ctx();
        c->device = device;
        c->sm_count = prop.multiProcessorCount;
        c->max_smem_optin = prop.sharedMemPerBlockOptin;
        LANE_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->error_flag = static_cast<int*>(dev_alloc(sizeof(int)));
        LANE_CUDA(cudaMemsetAsync(c->error_flag, 0, sizeof(int), c->stream));
        if (const char* e = std::getenv("LANE_B200_NUMERICS"))
            c->numerics = std::strcmp(e, "strict") == 0 ? LANE_NUMERICS_STRICT : LANE_NUMERICS_FAST;
        *out = c;
    });
}

static void release_ctx(lane_b200_ctx* c) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    comm_destroy(c->comm);
    for (void* p : c->scratch) cudaFree(p);
    cudaFree(c->error_flag);
    cudaStreamDestroy(c->stream);
    delete c;
}

int lane_b200_ctx_destroy(lane_b200_ctx* c) {
    return guard([&] {
        if (!c) return;
        if (c->live_nets > 0) {
            c->destroy_requested = true;  // released by the last net_destroy
            return;
        }
        release_ctx(c);
    });
}

int lane_b200_ctx_set_numerics(lane_b200_ctx* c, int mode) {
    return guard([&] {
        if (!c || (mode != LANE_NUMERICS_STRICT && mode != LANE_NUMERICS_FAST))
            throw Error(LANE_ERR_CONFIG, "bad numerics mode");
        c->numerics = mode;
    });
}

int lane_b200_ctx_get_numerics(lane_b200_ctx* c, int* mode) {
    return guard([&] {
        if (!c || !mode) throw Error(LANE_ERR_CONFIG, "null argument");
        *mode = c->numerics;
    });
}

int lane_b200_sync(lane_b200_ctx* c) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        c->check_device_error();
    });
}

int lane_b200_ctx_stream(lane_b200_ctx* c, void** stream) {
    return guard([&] {
        if (!c || !stream) throw Error(LANE_ERR_CONFIG, "null argument");
        *stream = c->stream;
    });
}

int lane_b200_kernel_launches(lane_b200_ctx* c, uint64_t* count) {
    return guard([&] {
        if (!c || !count) throw Error(LANE_ERR_CONFIG, "null argument");
        *count = c->launches;
    });
}

int lane_b200_dev_alloc(lane_b200_ctx* c, size_t bytes, void** dev) {
    return guard([&] {
        if (!c || !dev) throw Error(LANE_ERR_CONFIG, "null argument");
        LANE_CUDA(cudaSetDevice(c->device));
        *dev = dev_alloc(bytes);
        c->scratch.push_back(*dev);
    });
}

int lane_b200_dev_free(lane_b200_ctx* c, void* dev) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        auto it = std::find(c->scratch.begin(), c->scratch.end(), dev);
        if (it == c->scratch.end()) throw Error(LANE_ERR_CONFIG, "pointer not owned by context");
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        LANE_CUDA(cudaFree(dev));
        c->scratch.erase(it);
    });
}

int lane_b200_memcpy_h2d(lane_b200_ctx* c, void* dev, const void* host, size_t bytes) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        LANE_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c->stream));
    });
}

int lane_b200_memcpy_d2h(lane_b200_ctx* c, void* host, const void* dev, size_t bytes) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        LANE_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
        LANE_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ---------------------------------------------------------------- net ---

int lane_b200_net_create(lane_b200_ctx* c, size_t input_width, const size_t* hidden, size_t n_hidden,
                         size_t classes, size_t max_batch, lane_b200_net** out) {
    return guard([&] {
        if (!c || !out) throw Error(LANE_ERR_CONFIG, "null argument");
        // FeedForwardNetwork ctor validation (network.cpp:28-42)
        if (input_width == 0) throw Error(LANE_ERR_CONFIG, "network: input_width must be >= 1");
        if (classes < 2) throw Error(LANE_ERR_CONFIG, "network: need at least 2 classes");
        for (size_t l = 0; l < n_hidden; ++l)
            if (hidden[l] == 0) throw Error(LANE_ERR_CONFIG, "network: hidden layer size must be >= 1");
        if (max_batch == 0) throw Error(LANE_ERR_CONFIG, "network: max_batch must be >= 1");
        LANE_CUDA(cudaSetDevice(c->device));
        if (c->destroy_requested) throw Error(LANE_ERR_CONFIG, "context is being destroyed");
        auto* net = new lane_b200_net();
        net->ctx = c;
        net->input_width = input_width;
        net->n_hidden = n_hidden;
        net->classes = classes;
        net->max_batch = max_batch;
        size_t w = input_width;
        for (size_t l = 0; l <= n_hidden; ++l) {
            LayerBufs Ly;
            Ly.I = w;
            Ly.O = l < n_hidden ? hidden[l] : classes;
            w = Ly.O;
            net->layers.push_back(Ly);
        }
        // arena: params | grads | DW,db | per-sample vectors (x B rows)
        auto pad = [](size_t n) { return (n + 63) & ~size_t(63); };  // 256-byte pieces
        size_t off = 0;
        std::vector<size_t> offs;
        for (auto& Ly : net->layers) {
            Ly.cnt[LANE_BUF_W] = Ly.cnt[LANE_BUF_G] = Ly.cnt[LANE_BUF_DW] = Ly.I * Ly.O;
            Ly.cnt[LANE_BUF_B] = Ly.cnt[LANE_BUF_NETIN] = Ly.cnt[LANE_BUF_OUTPUTS] = Ly.cnt[LANE_BUF_DELTAS] =
                Ly.cnt[LANE_BUF_DELTA_BIASES] = Ly.cnt[LANE_BUF_BIAS_GRAD] = Ly.O;
            Ly.cnt[LANE_BUF_INPUTS] = Ly.I;
        }
        size_t params_begin = off;
        for (auto& Ly : net->layers) {
            offs.push_back(off); off += pad(Ly.I * Ly.O);  // W
            offs.push_back(off); off += pad(Ly.O);         // b
        }
        net->params_count = off - params_begin;
        size_t grads_begin = off;
        for (auto& Ly : net->layers) {
            offs.push_back(off); off += pad(Ly.I * Ly.O);  // G
            offs.push_back(off); off += pad(Ly.O);         // bias grad
        }
        net->grads_count = off - grads_begin;
        for (auto& Ly : net->layers) {
            offs.push_back(off); off += pad(Ly.I * Ly.O);  // DW
            offs.push_back(off); off += pad(Ly.O);         // db
        }
        for (auto& Ly : net->layers) {
            offs.push_back(off); off += pad(Ly.I * max_batch);  // inputs
            offs.push_back(off); off += pad(Ly.O * max_batch);  // netin
            offs.push_back(off); off += pad(Ly.O * max_batch);  // outputs
            offs.push_back(off); off += pad(Ly.O * max_batch);  // deltas
        }
        size_t stage_off = off;
        off += pad(classes * max_batch);
        net->arena_bytes = off * sizeof(float);
        net->arena = static_cast<char*>(dev_alloc(net->arena_bytes));
        LANE_CUDA(cudaMemsetAsync(net->arena, 0, net->arena_bytes, c->stream));
        float* base = reinterpret_cast<float*>(net->arena);
        size_t k = 0;
        for (auto& Ly : net->layers) { Ly.buf[LANE_BUF_W] = base + offs[k++]; Ly.buf[LANE_BUF_B] = base + offs[k++]; }
        for (auto& Ly : net->layers) { Ly.buf[LANE_BUF_G] = base + offs[k++]; Ly.buf[LANE_BUF_BIAS_GRAD] = base + offs[k++]; }
        for (auto& Ly : net->layers) { Ly.buf[LANE_BUF_DW] = base + offs[k++]; Ly.buf[LANE_BUF_DELTA_BIASES] = base + offs[k++]; }
        for (auto& Ly : net->layers) {
            Ly.buf[LANE_BUF_INPUTS] = base + offs[k++];
            Ly.buf[LANE_BUF_NETIN] = base + offs[k++];
            Ly.buf[LANE_BUF_OUTPUTS] = base + offs[k++];
            Ly.buf[LANE_BUF_DELTAS] = base + offs[k++];
        }
        net->params = base + params_begin;
        net->grads = base + grads_begin;
        net->target_stage = base + stage_off;
        net->step = static_cast<long long*>(dev_alloc(sizeof(long long)));
        // loss sum and hit count side by side: one memset and one D2H per epoch
        net->loss_dev = static_cast<double*>(dev_alloc(2 * sizeof(double)));
        net->correct_dev = reinterpret_cast<unsigned long long*>(net->loss_dev + 1);
        // split-K partials of the FAST forward (sized up front: the forward is
        // also captured into CUDA graphs, where allocation is not allowed)
        size_t part = 0;
        for (auto& Ly : net->layers) part = std::max(part, (2 * (size_t)c->sm_count + (Ly.O + 31) / 32) * 32);
        ensure(net->scratch, net->scratch_count, part);
        c->live_nets++;
        *out = net;
    });
}

int lane_b200_net_init_seeded(lane_b200_net* net, uint64_t seed) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        // build_network (network.cpp:55-66): hidden layers in order, then output
        SplitMix64 rng(seed);
        std::vector<float> host;
        for (auto& Ly : net->layers) {
            host.resize(Ly.I * Ly.O);
            const float bound = 1.0f / std::sqrt(static_cast<float>(Ly.I));
            for (float& v : host) v = rng.uniform(-bound, bound);
            LANE_CUDA(cudaMemcpyAsync(Ly.buf[LANE_BUF_W], host.data(), host.size() * sizeof(float),
                                      cudaMemcpyHostToDevice, net->ctx->stream));
            LANE_CUDA(cudaMemsetAsync(Ly.buf[LANE_BUF_B], 0, Ly.O * sizeof(float), net->ctx->stream));
            LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));
        }
    });
}

int lane_b200_net_destroy(lane_b200_net* net) {
    return guard([&] {
        if (!net) return;
        cudaSetDevice(net->ctx->device);
        cudaStreamSynchronize(net->ctx->stream);
        minibatch_free(net->mb);
        if (net->nvls.bound) {
            nvls_release(net->nvls);  // the arena lives in the NVLS mapping
        } else {
            if (net->nvls.mc) nvls_release(net->nvls);
            cudaFree(net->arena);
        }
        cudaFree(net->scratch);
        cudaFree(net->step);
        cudaFree(net->loss_dev);
        cudaFree(net->slots);
        cudaFree(net->win_coef);
        cudaFree(net->win_ring);
        net->mb_graph.reset();
        net->pipe.release();
        for (cudaEvent_t e : net->plan_events) cudaEventDestroy(e);
        cudaFree(net->eval_buf);
        cudaFree(net->eval_ws);
        cudaFree(net->spec_dev);
        cudaFree(net->spec_stats);
        cudaFree(net->spec_snap);
        if (net->spec_host) cudaFreeHost(net->spec_host);
        cudaFree(net->eval_counters);
        cudaFree(net->data);
        cudaFree(net->order);
        lane_b200_ctx* c = net->ctx;
        delete net;
        if (--c->live_nets == 0 && c->destroy_requested) release_ctx(c);
    });
}

int lane_b200_net_shape(lane_b200_net* net, size_t layer, size_t* ci, size_t* co) {
    return guard([&] {
        check_layer(net, layer);
        if (ci) *ci = net->L(layer).I;
        if (co) *co = net->L(layer).O;
    });
}

int lane_b200_net_n_layers(lane_b200_net* net, size_t* n) {
    return guard([&] {
        if (!net || !n) throw Error(LANE_ERR_CONFIG, "null argument");
        *n = net->layers.size();
    });
}

int lane_b200_buf_read(lane_b200_net* net, size_t layer, int buf, float* host, size_t count) {
    return guard([&] {
        check_layer(net, layer);
        if (buf < 0 || buf >= LANE_BUF_COUNT) throw Error(LANE_ERR_CONFIG, "bad buffer id");
        LayerBufs& Ly = net->L(layer);
        if (count != Ly.cnt[buf]) throw Error(LANE_ERR_SHAPE, "buf_read: count mismatch");
        LANE_CUDA(cudaMemcpyAsync(host, Ly.buf[buf], count * sizeof(float), cudaMemcpyDeviceToHost,
                                  net->ctx->stream));
        LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));
        net->ctx->check_device_error();
    });
}

int lane_b200_buf_write(lane_b200_net* net, size_t layer, int buf, const float* host, size_t count) {
    return guard([&] {
        check_layer(net, layer);
        if (buf < 0 || buf >= LANE_BUF_COUNT) throw Error(LANE_ERR_CONFIG, "bad buffer id");
        LayerBufs& Ly = net->L(layer);
        if (count != Ly.cnt[buf]) throw Error(LANE_ERR_SHAPE, "buf_write: count mismatch");
        LANE_CUDA(cudaMemcpyAsync(Ly.buf[buf], host, count * sizeof(float), cudaMemcpyHostToDevice,
                                  net->ctx->stream));
        LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));
    });
}

int lane_b200_buf_device_ptr(lane_b200_net* net, size_t layer, int buf, float** dev, size_t* count) {
    return guard([&] {
        check_layer(net, layer);
        if (buf < 0 || buf >= LANE_BUF_COUNT) throw Error(LANE_ERR_CONFIG, "bad buffer id");
        if (dev) *dev = net->L(layer).buf[buf];
        if (count) *count = net->L(layer).cnt[buf];
    });
}

int lane_b200_net_hash(lane_b200_net* net, uint64_t* hash) {
    return guard([&] {
        if (!net || !hash) throw Error(LANE_ERR_CONFIG, "null argument");
        uint64_t h = 0xcbf29ce484222325ULL;
        std::vector<float> host;
        for (auto& Ly : net->layers) {
            for (int b : {LANE_BUF_W, LANE_BUF_B}) {
                host.resize(Ly.cnt[b]);
                LANE_CUDA(cudaMemcpyAsync(host.data(), Ly.buf[b], host.size() * sizeof(float),
                                          cudaMemcpyDeviceToHost, net->ctx->stream));
                LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));
                h = fnv1a64(host.data(), host.size() * sizeof(float), h);
            }
        }
        net->ctx->check_device_error();
        *hash = h;
    });
}

// ---------------------------------------------------------- layer API ---

int lane_b200_layer_forward(lane_b200_net* net, size_t layer, const float* x_host, size_t len) {
    return guard([&] {
        check_layer(net, layer);
        LayerBufs& Ly = net->L(layer);
        const float* src;
        if (x_host) {
            // compute_netin (layers.cpp:28-31)
            if (len != Ly.I)
                throw Error(LANE_ERR_SHAPE, "forward: input length " + std::to_string(len) +
                                                " != cols_input " + std::to_string(Ly.I));
            LANE_CUDA(cudaMemcpyAsync(Ly.buf[LANE_BUF_INPUTS], x_host, len * sizeof(float),
                                      cudaMemcpyHostToDevice, net->ctx->stream));
            src = Ly.buf[LANE_BUF_INPUTS];
        } else {
            if (layer == 0) throw Error(LANE_ERR_CONFIG, "forward: layer 0 needs an input vector");
            src = net->L(layer - 1).buf[LANE_BUF_OUTPUTS];
        }
        run_layer_forward(net, layer, src);
    });
}

int lane_b200_fc_backward(lane_b200_net* net, size_t layer, const float* nW_host, size_t rows,
                          size_t cols, const float* nd_host, size_t nd_len, float eta) {
    return guard([&] {
        check_layer(net, layer);
        check_eta(eta);
        if (layer >= net->n_hidden) throw Error(LANE_ERR_CONFIG, "fc_backward: not a hidden layer");
        LayerBufs& Ly = net->L(layer);
        const float* nW;
        const float* nd;
        size_t N;
        if (nW_host) {
            // FullyConnectedLayer::backward shape checks (layers.cpp:53-58)
            if (rows != Ly.O) throw Error(LANE_ERR_SHAPE, "fc backward: next_weights.rows != cols_out");
            if (nd_len != cols) throw Error(LANE_ERR_SHAPE, "fc backward: next_deltas length != next_weights.cols");
            ensure(net->scratch, net->scratch_count, rows * cols + cols);
            LANE_CUDA(cudaMemcpyAsync(net->scratch, nW_host, rows * cols * sizeof(float),
                                      cudaMemcpyHostToDevice, net->ctx->stream));
            LANE_CUDA(cudaMemcpyAsync(net->scratch + rows * cols, nd_host, cols * sizeof(float),
                                      cudaMemcpyHostToDevice, net->ctx->stream));
            nW = net->scratch;
            nd = net->scratch + rows * cols;
            N = cols;
        } else {
            LayerBufs& nx = net->L(layer + 1);
            nW = nx.buf[LANE_BUF_W];
            nd = nx.buf[LANE_BUF_DELTAS];
            N = nx.O;
        }
        run_fc_backward(net, layer, nW, nd, static_cast<int>(N), eta);
        if (nW_host) LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));  // scratch reuse
    });
}

int lane_b200_softmax_backward(lane_b200_net* net, const float* t_host, size_t len, float eta) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        check_eta(eta);
        // SoftmaxOutputLayer::backward (layers.cpp:90-92)
        if (len != net->classes) throw Error(LANE_ERR_SHAPE, "softmax backward: target length != cols_out");
        LANE_CUDA(cudaMemcpyAsync(net->target_stage, t_host, len * sizeof(float), cudaMemcpyHostToDevice,
                                  net->ctx->stream));
        run_softmax_backward(net, net->target_stage, eta);
    });
}

int lane_b200_apply_updates(lane_b200_net* net, size_t layer) {
    return guard([&] {
        check_layer(net, layer);
        run_apply_updates(net, layer);
    });
}

// -------------------------------------------------------- network API ---

int lane_b200_forward(lane_b200_net* net, const float* x_host, float* probs_host) {
    return guard([&] {
        if (!net || !x_host) throw Error(LANE_ERR_CONFIG, "null argument");
        LANE_CUDA(cudaMemcpyAsync(net->L(0).buf[LANE_BUF_INPUTS], x_host, net->input_width * sizeof(float),
                                  cudaMemcpyHostToDevice, net->ctx->stream));
        run_forward_chain(net);
        if (probs_host) {
            LANE_CUDA(cudaMemcpyAsync(probs_host, net->L(net->out_layer()).buf[LANE_BUF_OUTPUTS],
                                      net->classes * sizeof(float), cudaMemcpyDeviceToHost, net->ctx->stream));
            LANE_CUDA(cudaStreamSynchronize(net->ctx->stream));
        }
    });
}

int lane_b200_backward_plan_run(lane_b200_net* net, const float* t_host, float eta) {
    return guard([&] {
        if (!net || !t_host) throw Error(LANE_ERR_CONFIG, "null argument");
        check_eta(eta);
        LANE_CUDA(cudaMemcpyAsync(net->target_stage, t_host, net->classes * sizeof(float),
                                  cudaMemcpyHostToDevice, net->ctx->stream));
        run_backward_plan(net, net->target_stage, eta);
    });
}

int lane_b200_backward_plan_run_timed(lane_b200_net* net, const float* t_host, float eta, double* phase_ms,
                                      size_t n_phase) {
    return guard([&] {
        if (!net || !t_host || !phase_ms) throw Error(LANE_ERR_CONFIG, "null argument");
        check_eta(eta);
        const size_t nl = net->layers.size();
        if (n_phase < 3 * nl) throw Error(LANE_ERR_SHAPE, "backward_plan_run_timed: phase_ms too short");
        cudaStream_t st = net->ctx->stream;
        // events: [0] start, [1] target uploaded, [2 + k] end of schedule k
        std::vector<cudaEvent_t>& ev = net->plan_events;
        while (ev.size() < nl + 2) {
            cudaEvent_t e;
            LANE_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
        }
        LANE_CUDA(cudaEventRecord(ev[0], st));
        LANE_CUDA(cudaMemcpyAsync(net->target_stage, t_host, net->classes * sizeof(float), cudaMemcpyHostToDevice,
                                  st));
        LANE_CUDA(cudaEventRecord(ev[1], st));
        run_softmax_backward(net, net->target_stage, eta);
        LANE_CUDA(cudaEventRecord(ev[2], st));
        size_t k = 1;
        for (size_t l = net->n_hidden; l-- > 0; ++k) {
            LayerBufs& nx = net->L(l + 1);
            run_fc_backward(net, l, nx.buf[LANE_BUF_W], nx.buf[LANE_BUF_DELTAS], static_cast<int>(nx.O), eta);
            LANE_CUDA(cudaEventRecord(ev[2 + k], st));
        }
        for (size_t l = 0; l < nl; ++l) run_apply_updates(net, l);
        LANE_CUDA(cudaEventSynchronize(ev[1 + nl]));
        float ms = 0.0f;
        LANE_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        phase_ms[0] = ms;
        LANE_CUDA(cudaEventElapsedTime(&ms, ev[1], ev[2]));
        phase_ms[1] = ms;
        phase_ms[2] = 0.0;
        for (size_t j = 1; j < nl; ++j) {
            LANE_CUDA(cudaEventElapsedTime(&ms, ev[1 + j], ev[2 + j]));
            phase_ms[3 * j + 0] = 0.0;
            phase_ms[3 * j + 1] = ms;
            phase_ms[3 * j + 2] = 0.0;
        }
        LANE_CUDA(cudaStreamSynchronize(st));
    });
}

int lane_b200_sgd_stream(lane_b200_net* net, const float* X, const float* T, size_t n, const uint32_t* order,
                         size_t n_steps, float eta, double* loss_sum, uint64_t* correct) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        sgd_stream_impl(net, X, T, n, order, n_steps, eta, loss_sum,
                        reinterpret_cast<unsigned long long*>(correct));
    });
}

int lane_b200_sgd_stream_plan(lane_b200_net* net, char* buf, size_t len) {
    return guard([&] {
        if (!net || !buf || len == 0) throw Error(LANE_ERR_CONFIG, "null argument");
        const SgdPlan P = plan_persistent(net);
        char tmp[128];
        if (tiny_plan(net))
            std::snprintf(tmp, sizeof tmp, "tiny one warp, reference arithmetic");
        else if (!P.ok)
            std::snprintf(tmp, sizeof tmp, "layer");
        else if (P.window)
            std::snprintf(tmp, sizeof tmp, "window D=%d KS=%d QPC=%d chain=%dx%dx%d ctas=%d smem=%zu", P.D, P.ks,
                          P.qpc, P.cs, P.ncw, 32 * P.jpl, P.G, P.smem);
        else if (P.cluster)
            std::snprintf(tmp, sizeof tmp, "cluster ctas=%d smem=%zu", P.G, P.smem);
        else
            std::snprintf(tmp, sizeof tmp, "grid ctas=%d w0=%s smem=%zu", P.G, P.w0_smem ? "smem" : "hbm", P.smem);
        std::snprintf(buf, len, "%s", tmp);
    });
}

int lane_b200_train(lane_b200_net* net, const float* X_host, const float* T_host, size_t n, float eta,
                    float max_error, size_t max_epochs, uint64_t seed, float* mean_loss_out,
                    float* accuracy_out, size_t* epochs_run) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        check_eta(eta);
        // train (network.cpp:142-150)
        if (n == 0) throw Error(LANE_ERR_TRAINING, "train: empty training set");
        if (n > 0xffffffffull) throw Error(LANE_ERR_SHAPE, "train: more than 2^32 samples");
        lane_b200_ctx* c = net->ctx;
        const size_t I = net->input_width, C = net->classes;
        // The epoch streams through the input pipeline (pipeline.cuh) in
        // chunks of consecutive stream positions: the host gathers the rows of
        // the epoch's permutation into a page-locked slot, the copy stream
        // uploads it, and the fused kernel runs the chunk as a contiguous
        // stream -- the upload of chunk k+1 overlaps the kernel on chunk k.
        // Chunks start small (little exposed copy) and double.
        constexpr size_t kFirst = 512, kMax = 16384;
        InputPipeline& P = net->pipe;
        SplitMix64 shuffle(seed);  // one generator for the whole run (network.cpp:153)
        std::vector<uint32_t> order(n);
        for (size_t k = 0; k < n; ++k) order[k] = static_cast<uint32_t>(k);
        size_t ran = 0, done = 0;
        // Small sets (C1's 135-sample Iris epochs run in ~90 us) are bound by the
        // per-epoch host round trip, not by the kernel.  Epochs then run
        // speculatively in batches of K (2, doubling to 32) with no host sync
        // in between: each epoch accumulates into its own stats slot, and the
        // arena (weights, gradients, deltas, per-sample vectors) is snapshotted
        // after every epoch but the batch's last.  One read-back per batch finds
        // the first epoch with mean_loss <= max_error; the arena is restored to
        // the snapshot after it, so the result is bitwise the epoch-by-epoch
        // run's (train's stop rule, network.cpp:173-181).
        constexpr size_t kSpecMax = 32;
        if (n <= kMax && net->arena_bytes <= (size_t(8) << 20) && std::getenv("LANE_B200_TRAIN_NOSPEC") == nullptr) {
            // per epoch: X rows then T rows, each piece 256-byte aligned (the
            // kernels read rows with 16-byte vector loads)
            const size_t xoff = (n * I + 63) & ~size_t(63);
            const size_t row = xoff + ((n * C + 63) & ~size_t(63));
            ensure(net->spec_dev, net->spec_dev_count, kSpecMax * row);
            ensure(net->spec_stats, net->spec_stats_count, 4 * kSpecMax);  // doubles
            ensure(net->spec_snap, net->spec_snap_count, (kSpecMax - 1) * net->arena_bytes / sizeof(float) + 64);
            if (net->spec_host_count < kSpecMax * row) {
                if (net->spec_host) LANE_CUDA(cudaFreeHost(net->spec_host));
                net->spec_host = nullptr;
                LANE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&net->spec_host), kSpecMax * row * sizeof(float),
                                        cudaHostAllocDefault));
                net->spec_host_count = kSpecMax * row;
            }
            double* stats_dev = reinterpret_cast<double*>(net->spec_stats);
            char* snaps = reinterpret_cast<char*>(net->spec_snap);
            std::vector<double> stats(2 * kSpecMax);
            size_t K = 2;
            while (ran < max_epochs) {
                const size_t k_run = std::min(K, max_epochs - ran);
                for (size_t e = 0; e < k_run; ++e) {
                    for (size_t i = n; i > 1; --i) std::swap(order[i - 1], order[shuffle.below(i)]);
                    gather_rows(X_host, T_host, I, C, order.data(), n, net->spec_host + e * row);
                    // gather_rows packs T right after X: move it to its aligned offset
                    float* h = net->spec_host + e * row;
                    if (xoff != n * I) std::memmove(h + xoff, h + n * I, n * C * sizeof(float));
                }
                LANE_CUDA(cudaMemcpyAsync(net->spec_dev, net->spec_host, k_run * row * sizeof(float),
                                          cudaMemcpyHostToDevice, c->stream));
                LANE_CUDA(cudaMemsetAsync(stats_dev, 0, 2 * k_run * sizeof(double), c->stream));
                for (size_t e = 0; e < k_run; ++e) {
                    const float* Xd = net->spec_dev + e * row;
                    sgd_stream_impl(net, Xd, Xd + xoff, n, nullptr, n, eta, stats_dev + 2 * e,
                                    reinterpret_cast<unsigned long long*>(stats_dev + 2 * e + 1));
                    if (e + 1 < k_run)
                        LANE_CUDA(cudaMemcpyAsync(snaps + e * net->arena_bytes, net->arena, net->arena_bytes,
                                                  cudaMemcpyDeviceToDevice, c->stream));
                }
                int dev_err = 0;
                LANE_CUDA(cudaMemcpyAsync(stats.data(), stats_dev, 2 * k_run * sizeof(double), cudaMemcpyDeviceToHost,
                                          c->stream));
                LANE_CUDA(cudaMemcpyAsync(&dev_err, c->error_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
                LANE_CUDA(cudaStreamSynchronize(c->stream));
                if (dev_err) c->check_device_error();
                bool stop = false;
                for (size_t e = 0; e < k_run && !stop; ++e) {
                    unsigned long long correct = 0;
                    std::memcpy(&correct, &stats[2 * e + 1], sizeof(correct));
                    const float mean_loss = static_cast<float>(stats[2 * e] / static_cast<double>(n));
                    if (mean_loss_out) mean_loss_out[ran] = mean_loss;
                    if (accuracy_out) accuracy_out[ran] = static_cast<float>(correct) / static_cast<float>(n);
                    ++ran;
                    if (mean_loss <= max_error) {
                        stop = true;
                        if (e + 1 < k_run)  // roll the speculative epochs back
                            LANE_CUDA(cudaMemcpyAsync(net->arena, snaps + e * net->arena_bytes, net->arena_bytes,
                                                      cudaMemcpyDeviceToDevice, c->stream));
                    }
                }
                if (stop) break;
                K = std::min(2 * K, kSpecMax);
            }
            LANE_CUDA(cudaStreamSynchronize(c->stream));
            if (epochs_run) *epochs_run = ran;
            return;
        }
        P.reserve(std::min(n, kMax) * (I + C), 1);
        for (size_t epoch = 1; epoch <= max_epochs; ++epoch) {
            for (size_t i = n; i > 1; --i) std::swap(order[i - 1], order[shuffle.below(i)]);
            LANE_CUDA(cudaMemsetAsync(net->loss_dev, 0, 2 * sizeof(double), c->stream));  // loss + hits
            size_t chunk = kFirst;
            for (size_t s = 0; s < n; s += chunk, chunk = std::min(2 * chunk, kMax)) {
                const size_t m = std::min(chunk, n - s);
                const int k = static_cast<int>(done++ % InputPipeline::kSlots);
                if (P.pending[k]) LANE_CUDA(cudaEventSynchronize(P.copied[k]));
                gather_rows(X_host, T_host, I, C, order.data() + s, m, P.host[k]);
                if (m == n) {
                    // the whole epoch in one chunk: nothing to overlap, so copy on
                    // the compute stream (no cross-stream events on the latency path)
                    LANE_CUDA(cudaMemcpyAsync(P.dev[k], P.host[k], m * (I + C) * sizeof(float),
                                              cudaMemcpyHostToDevice, c->stream));
                    LANE_CUDA(cudaEventRecord(P.copied[k], c->stream));
                } else {
                    LANE_CUDA(cudaStreamWaitEvent(P.copy, P.consumed[k], 0));
                    LANE_CUDA(cudaMemcpyAsync(P.dev[k], P.host[k], m * (I + C) * sizeof(float),
                                              cudaMemcpyHostToDevice, P.copy));
                    LANE_CUDA(cudaEventRecord(P.copied[k], P.copy));
                    LANE_CUDA(cudaStreamWaitEvent(c->stream, P.copied[k], 0));
                }
                sgd_stream_impl(net, P.dev[k], P.dev[k] + m * I, m, nullptr, m, eta, net->loss_dev,
                                net->correct_dev);
                LANE_CUDA(cudaEventRecord(P.consumed[k], c->stream));
                P.pending[k] = true;
            }
            double stats[2];  // loss sum, hit count (bit pattern)
            int dev_err = 0;  // persistent-kernel exchange timeout flag, read in the same round trip
            LANE_CUDA(cudaMemcpyAsync(stats, net->loss_dev, sizeof(stats), cudaMemcpyDeviceToHost, c->stream));
            LANE_CUDA(cudaMemcpyAsync(&dev_err, c->error_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            LANE_CUDA(cudaStreamSynchronize(c->stream));
            if (dev_err) c->check_device_error();  // resets the flag and throws
            const double loss_sum = stats[0];
            unsigned long long correct = 0;
            std::memcpy(&correct, &stats[1], sizeof(correct));
            const float mean_loss = static_cast<float>(loss_sum / static_cast<double>(n));
            const float acc = static_cast<float>(correct) / static_cast<float>(n);
            if (mean_loss_out) mean_loss_out[ran] = mean_loss;
            if (accuracy_out) accuracy_out[ran] = acc;
            ++ran;
            if (mean_loss <= max_error) break;
        }
        if (epochs_run) *epochs_run = ran;
    });
}

}  // extern "C"

namespace {

// evaluate in FAST numerics: the forward of whole row chunks as GEMMs (the
// mini-batch path's kernels: tcgen05 3xTF32 where eligible, bias/tanh fused),
// then per-row softmax / cross entropy / argmax and one fixed-order reduction.
// STRICT evaluation keeps the per-sample layer path (bit-exact).
void evaluate_batched(lane_b200_net* net, const float* Xd, const float* Td, size_t n) {
    lane_b200_ctx* c = net->ctx;
    const int nl = static_cast<int>(net->layers.size());
    const int C = static_cast<int>(net->classes);
    size_t wmax = net->classes;
    for (auto& Ly : net->layers) wmax = std::max(wmax, Ly.O);
    const size_t R = std::min<size_t>(n, 8192);
    // scratch: z | a0 | a1 (R x wmax each) | row losses | row hits
    ensure(net->eval_buf, net->eval_count, 3 * R * wmax + 2 * R + 64);
    float* z = net->eval_buf;
    float* act[2] = {z + R * wmax, z + 2 * R * wmax};
    float* row_loss = z + 3 * R * wmax;
    float* row_ok = row_loss + R;
    // its own GEMM workspace: the mini-batch step graph holds net->mb.ws
    GemmCtx g{c->stream,      c->sm_count, &net->eval_ws, &net->eval_ws_count, &c->launches, nullptr,
              &net->eval_counters, &net->eval_counters_count};
    for (size_t r0 = 0; r0 < n; r0 += R) {
        const int rows = static_cast<int>(std::min(R, n - r0));
        const float* in = Xd + r0 * net->input_width;
        for (int l = 0; l < nl; ++l) {
            LayerBufs& Ly = net->L(l);
            const bool last = l == nl - 1;
            float* out = act[l & 1];
            gemm(g, GemmOp::NN, rows, (int)Ly.O, (int)Ly.I, in, (int)Ly.I, Ly.buf[LANE_BUF_W], (int)Ly.O,
                 last ? Epi::BIAS : Epi::BIAS_TANH, z, last ? nullptr : out, Ly.buf[LANE_BUF_B], nullptr);
            in = out;
        }
        k_eval_rows<<<(rows + 127) / 128, 128, 0, c->stream>>>(z, Td + r0 * C, rows, C, row_loss, row_ok);
        k_eval_reduce<<<1, 32, 0, c->stream>>>(row_loss, row_ok, rows, net->loss_dev, net->correct_dev);
        c->count(2);
    }
    c->check_launch();
}

}  // namespace

extern "C" {

int lane_b200_evaluate(lane_b200_net* net, const float* X_host, const float* T_host, size_t n, float* mean_loss,
                       float* accuracy) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        // evaluate (network.cpp:186-191)
        if (n == 0) throw Error(LANE_ERR_TRAINING, "evaluate: empty test set");
        lane_b200_ctx* c = net->ctx;
        const size_t I = net->input_width, C = net->classes;
        ensure(net->data, net->data_count, n * (I + C));
        float* Xd = net->data;
        float* Td = net->data + n * I;
        LANE_CUDA(cudaMemcpyAsync(Xd, X_host, n * I * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        LANE_CUDA(cudaMemcpyAsync(Td, T_host, n * C * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        LANE_CUDA(cudaMemsetAsync(net->loss_dev, 0, sizeof(double), c->stream));
        LANE_CUDA(cudaMemsetAsync(net->correct_dev, 0, sizeof(unsigned long long), c->stream));
        if (c->numerics == LANE_NUMERICS_STRICT || n < 64 || C > 128)
            stream_layer_path(net, Xd, Td, n, nullptr, n, 1.0f, net->loss_dev, net->correct_dev, false);
        else
            evaluate_batched(net, Xd, Td, n);
        double loss_sum = 0;
        unsigned long long correct = 0;
        LANE_CUDA(cudaMemcpyAsync(&loss_sum, net->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        LANE_CUDA(cudaMemcpyAsync(&correct, net->correct_dev, sizeof(correct), cudaMemcpyDeviceToHost, c->stream));
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        if (mean_loss) *mean_loss = static_cast<float>(loss_sum / static_cast<double>(n));
        if (accuracy) *accuracy = static_cast<float>(correct) / static_cast<float>(n);
    });
}

// ------------------------------------------------- mini-batch + comms ---

namespace {

void minibatch_step_impl(lane_b200_net* net, const float* X, const float* T, size_t B, float eta, float mu,
                         double* loss_sum) {
    lane_b200_ctx* c = net->ctx;
    minibatch_stage(*c, *net, X, T, B);
    // The step body runs eagerly once per configuration (sizing every
    // workspace), then as a captured CUDA graph: ~20 launches -> one.
    MbGraph& gr = net->mb_graph;
    const MbGraph::Key key{B,        eta,           mu, loss_sum, c->comm.world, c->numerics, gemm_tc_mode(),
                           static_cast<const void*>(c->comm.comm), net->mb.ws, net->mb.ws_gen};
    const bool use_graph = !std::getenv("LANE_B200_MB_NOGRAPH");
    if (use_graph && gr.exec && gr.key == key) {
        LANE_CUDA(cudaGraphLaunch(gr.exec, c->stream));
        c->count(static_cast<int>(gr.launches));
    } else if (use_graph && gr.warm && gr.key == key) {
        gr.reset();
        cudaGraph_t graph = nullptr;
        const uint64_t before = c->launches;
        LANE_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            minibatch_body(*c, *net, B, eta, mu, loss_sum);
        } catch (...) {
            cudaStreamEndCapture(c->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        LANE_CUDA(cudaStreamEndCapture(c->stream, &graph));
        gr.launches = c->launches - before;
        c->launches = before;
        LANE_CUDA(cudaGraphInstantiate(&gr.exec, graph, 0));
        LANE_CUDA(cudaGraphDestroy(graph));
        gr.key = key;
        LANE_CUDA(cudaGraphLaunch(gr.exec, c->stream));
        c->count(static_cast<int>(gr.launches));
    } else {
        gr.reset();
        minibatch_body(*c, *net, B, eta, mu, loss_sum);
        gr.key = key;
        gr.key.ws = net->mb.ws;  // the eager run sized the workspace
        gr.key.ws_gen = net->mb.ws_gen;
        gr.warm = true;
    }
    c->check_launch();
}

}  // namespace

int lane_b200_minibatch_step(lane_b200_net* net, const float* X, const float* T, size_t B, float eta, float mu,
                             double* loss_sum) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        check_eta(eta);
        check_mu(mu);
        if (B == 0 || B > net->max_batch) throw Error(LANE_ERR_SHAPE, "minibatch: B must be in [1, max_batch]");
        minibatch_step_impl(net, X, T, B, eta, mu, loss_sum);
    });
}

int lane_b200_minibatch_grads(lane_b200_net* net, const float* X, const float* T, size_t B, double* loss_sum) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        if (B == 0 || B > net->max_batch) throw Error(LANE_ERR_SHAPE, "minibatch: B must be in [1, max_batch]");
        minibatch_stage(*net->ctx, *net, X, T, B);
        minibatch_grads_body(*net->ctx, *net, B, loss_sum, false);
    });
}

int lane_b200_minibatch_apply(lane_b200_net* net, size_t B_global, float eta, float mu) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        check_eta(eta);
        check_mu(mu);
        if (B_global == 0) throw Error(LANE_ERR_SHAPE, "minibatch_apply: B_global must be >= 1");
        minibatch_update(*net->ctx, *net, B_global, eta, mu);
    });
}

int lane_b200_net_grads_arena(lane_b200_net* net, float** dev, size_t* count) {
    return guard([&] {
        if (!net || !dev || !count) throw Error(LANE_ERR_CONFIG, "null argument");
        *dev = net->grads;
        *count = net->grads_count;
    });
}

int lane_b200_train_minibatch(lane_b200_net* net, const float* X_host, const float* T_host, size_t n,
                              size_t batch, float eta, float mu, size_t epochs, uint64_t seed, int shuffle,
                              int drop_last, float* mean_loss_out, float* step_loss_out, size_t* steps_run) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        check_eta(eta);
        check_mu(mu);
        if (!X_host || !T_host) throw Error(LANE_ERR_CONFIG, "train_minibatch: null dataset");
        if (n == 0) throw Error(LANE_ERR_TRAINING, "train_minibatch: empty training set");
        if (batch == 0 || batch > net->max_batch)
            throw Error(LANE_ERR_SHAPE, "train_minibatch: batch must be in [1, max_batch]");
        if (n > 0xffffffffull) throw Error(LANE_ERR_SHAPE, "train_minibatch: more than 2^32 samples");
        lane_b200_ctx* c = net->ctx;
        const size_t I = net->input_width, C = net->classes;
        const int world = std::max(1, c->comm.world), rank = c->comm.rank;
        // rank r takes rows [r*batch, (r+1)*batch) of every global batch
        const size_t BG = batch * static_cast<size_t>(world);
        const size_t full = n / BG;
        const size_t tail = (world == 1 && !drop_last) ? n % BG : 0;
        const size_t steps = full + (tail ? 1 : 0);
        if (steps == 0) throw Error(LANE_ERR_TRAINING, "train_minibatch: fewer samples than one global batch");
        InputPipeline& P = net->pipe;
        // the running loss after every step of the whole call (epochs x steps,
        // pinned): one host synchronisation at the end instead of one per epoch,
        // so the pipeline never drains at an epoch boundary
        P.reserve(batch * (I + C), epochs * steps);
        // rows straight from page-locked dataset memory when a step's rows are
        // consecutive (no shuffle): no host gather, no staging copy
        cudaPointerAttributes ax{}, at{};
        const bool pinned_src = cudaPointerGetAttributes(&ax, X_host) == cudaSuccess &&
                                cudaPointerGetAttributes(&at, T_host) == cudaSuccess &&
                                ax.type == cudaMemoryTypeHost && at.type == cudaMemoryTypeHost;
        cudaGetLastError();  // a pageable pointer is not an error here
        std::vector<uint32_t> order(n);
        for (size_t k = 0; k < n; ++k) order[k] = static_cast<uint32_t>(k);
        SplitMix64 rng(seed);  // one generator for the whole run, like train (network.cpp:153)
        size_t done = 0;
        for (size_t epoch = 0; epoch < epochs; ++epoch) {
            // the permutation continues from the previous epoch's (network.cpp:154-161)
            if (shuffle)
                for (size_t i = n; i > 1; --i) std::swap(order[i - 1], order[rng.below(i)]);
            LANE_CUDA(cudaMemsetAsync(net->loss_dev, 0, sizeof(double), c->stream));
            for (size_t s = 0; s < steps; ++s) {
                const size_t rows = s < full ? batch : tail;
                const int k = static_cast<int>(done % InputPipeline::kSlots);
                const uint32_t* idx = order.data() + s * BG + (s < full ? rank * batch : 0);
                bool direct = pinned_src;
                for (size_t j = 1; direct && j < rows; ++j) direct = idx[j] == idx[0] + j;
                LANE_CUDA(cudaStreamWaitEvent(P.copy, P.consumed[k], 0));  // device slot free
                if (direct) {
                    LANE_CUDA(cudaMemcpyAsync(P.dev[k], X_host + static_cast<size_t>(idx[0]) * I,
                                              rows * I * sizeof(float), cudaMemcpyHostToDevice, P.copy));
                    LANE_CUDA(cudaMemcpyAsync(P.dev[k] + rows * I, T_host + static_cast<size_t>(idx[0]) * C,
                                              rows * C * sizeof(float), cudaMemcpyHostToDevice, P.copy));
                } else {
                    if (P.pending[k]) LANE_CUDA(cudaEventSynchronize(P.copied[k]));  // pinned slot free
                    gather_rows(X_host, T_host, I, C, idx, rows, P.host[k]);
                    LANE_CUDA(cudaMemcpyAsync(P.dev[k], P.host[k], rows * (I + C) * sizeof(float),
                                              cudaMemcpyHostToDevice, P.copy));
                }
                LANE_CUDA(cudaEventRecord(P.copied[k], P.copy));
                LANE_CUDA(cudaStreamWaitEvent(c->stream, P.copied[k], 0));
                minibatch_step_impl(net, P.dev[k], P.dev[k] + rows * I, rows, eta, mu, net->loss_dev);
                LANE_CUDA(cudaEventRecord(P.consumed[k], c->stream));
                P.pending[k] = true;
                // the step's result back to the host: the running loss sum (8 bytes, async)
                LANE_CUDA(cudaMemcpyAsync(P.cum_loss_host + done, net->loss_dev, sizeof(double),
                                          cudaMemcpyDeviceToHost, c->stream));
                ++done;
            }
        }
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        c->check_device_error();
        size_t local = 0;
        for (size_t s = 0; s < steps; ++s) local += s < full ? batch : tail;
        for (size_t epoch = 0; epoch < epochs; ++epoch) {
            const double* cum = P.cum_loss_host + epoch * steps;
            if (mean_loss_out) mean_loss_out[epoch] = static_cast<float>(cum[steps - 1] / static_cast<double>(local));
            if (step_loss_out)
                for (size_t s = 0; s < steps; ++s) {
                    const double prev = s ? cum[s - 1] : 0.0;
                    const size_t rows = s < full ? batch : tail;
                    step_loss_out[epoch * steps + s] = static_cast<float>((cum[s] - prev) / static_cast<double>(rows));
                }
        }
        if (steps_run) *steps_run = done;
    });
}

// ------------------------------------------------------------ datasets ---

int lane_b200_dataset_create(size_t features, size_t classes, size_t n, const float* X, const float* T,
                             lane_b200_dataset** out) {
    return guard([&] {
        if (!out || (n && (!X || !T))) throw Error(LANE_ERR_CONFIG, "null argument");
        auto d = std::make_unique<lane_b200_dataset>();
        d->allocate(features, classes, n);
        if (n) {
            std::memcpy(d->X, X, n * features * sizeof(float));
            std::memcpy(d->T, T, n * classes * sizeof(float));
        }
        *out = d.release();
    });
}

int lane_b200_dataset_load(const char* path, size_t features, size_t classes, lane_b200_dataset** out) {
    return guard([&] {
        if (!path || !out) throw Error(LANE_ERR_CONFIG, "null argument");
        auto d = std::make_unique<lane_b200_dataset>();
        lane_b200::dataset::load(path, features, classes, *d);
        *out = d.release();
    });
}

int lane_b200_dataset_save(const lane_b200_dataset* d, const char* path) {
    return guard([&] {
        if (!d || !path) throw Error(LANE_ERR_CONFIG, "null argument");
        lane_b200::dataset::save(*d, path);
    });
}

int lane_b200_dataset_info(const lane_b200_dataset* d, size_t* features, size_t* classes, size_t* n, float** X,
                           float** T, int* pinned) {
    return guard([&] {
        if (!d) throw Error(LANE_ERR_CONFIG, "null dataset");
        if (features) *features = d->features;
        if (classes) *classes = d->classes;
        if (n) *n = d->n;
        if (X) *X = d->X;
        if (T) *T = d->T;
        if (pinned) *pinned = d->pinned ? 1 : 0;
    });
}

int lane_b200_dataset_split(const lane_b200_dataset* d, double train_fraction, uint64_t seed,
                            lane_b200_dataset** train, lane_b200_dataset** test) {
    return guard([&] {
        if (!d || !train || !test) throw Error(LANE_ERR_CONFIG, "null argument");
        auto a = std::make_unique<lane_b200_dataset>();
        auto b = std::make_unique<lane_b200_dataset>();
        lane_b200::dataset::split(*d, train_fraction, seed, *a, *b);
        *train = a.release();
        *test = b.release();
    });
}

int lane_b200_dataset_enlarge(const lane_b200_dataset* d, size_t factor, float noise, uint64_t* rng_state,
                              lane_b200_dataset** out) {
    return guard([&] {
        if (!d || !rng_state || !out) throw Error(LANE_ERR_CONFIG, "null argument");
        auto e = std::make_unique<lane_b200_dataset>();
        lane_b200::dataset::enlarge(*d, factor, noise, *rng_state, *e);
        *out = e.release();
    });
}

int lane_b200_dataset_destroy(lane_b200_dataset* d) {
    return guard([&] { delete d; });
}
int lane_b200_gemm(lane_b200_ctx* c, int op, int M, int N, int K, const float* A, const float* B, float* C,
                   float* C2, const float* bias, const float* aux, int epilogue, int use_tc) {
    return lane_b200_gemm_ex(c, op, M, N, K, A, B, C, C2, bias, aux, epilogue, use_tc, nullptr, nullptr);
}

int lane_b200_absmax(lane_b200_ctx* c, const float* X, int rows, int cols, unsigned* row_max, unsigned* col_max) {
    return guard([&] {
        if (!c || !X || !row_max || !col_max || rows < 1 || cols < 4 || (cols & 3))
            throw Error(LANE_ERR_CONFIG, "lane_b200_absmax: bad arguments (cols a positive multiple of 4)");
        LANE_CUDA(cudaMemsetAsync(row_max, 0, (size_t)rows * sizeof(unsigned), c->stream));
        LANE_CUDA(cudaMemsetAsync(col_max, 0, (size_t)cols * sizeof(unsigned), c->stream));
        absmax_rc_launch(c->stream, X, rows, cols, row_max, col_max);
        c->count(1);
        c->check_launch();
    });
}

int lane_b200_gemm_ex(lane_b200_ctx* c, int op, int M, int N, int K, const float* A, const float* B, float* C,
                      float* C2, const float* bias, const float* aux, int epilogue, int use_tc, const unsigned* amax,
                      const unsigned* bmax) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        if (op < 0 || op > 2 || epilogue < 0 || epilogue > 3 || M < 0 || N < 0 || K < 0 || use_tc < 0 || use_tc > 5)
            throw Error(LANE_ERR_CONFIG, "lane_b200_gemm: bad op/epilogue/shape");
        static float* ws = nullptr;
        static size_t ws_count = 0;
        static int* counters = nullptr;
        static size_t counters_count = 0;
        GemmCtx g{c->stream, c->sm_count, &ws, &ws_count, &c->launches, nullptr, &counters, &counters_count};
        const GemmOp o = static_cast<GemmOp>(op);
        const int lda = o == GemmOp::TN ? M : K;
        const int ldb = o == GemmOp::NT ? K : N;
        const int saved = gemm_tc_mode(), saved_p = tc_persist_mode(), saved_h = tc_prec_mode();
        gemm_tc_mode() = use_tc ? 1 : 0;
        // 4: the 3xF16 kernel (gemm_h3.cuh); 5: the mini-batch step's own choice
        // (3xF16 for the tall long-K shapes); else 3xTF32
        tc_prec_mode() = use_tc == 4 ? 1 : use_tc == 5 ? saved_h : 0;
        if (use_tc == 2) tc_persist_mode() = 2;  // the persistent stream-K kernel for every shape
        if (use_tc == 3) tc_persist_mode() = 0;  // never
        try {
            GemmMax mx;
            mx.a = amax;
            mx.b = bmax;
            gemm(g, o, M, N, K, A, lda, B, ldb, static_cast<Epi>(epilogue), C, C2, bias, aux,
                 (amax && bmax) ? &mx : nullptr);
        } catch (...) {
            gemm_tc_mode() = saved;
            tc_persist_mode() = saved_p;
            tc_prec_mode() = saved_h;
            throw;
        }
        gemm_tc_mode() = saved;
        tc_persist_mode() = saved_p;
        tc_prec_mode() = saved_h;
        c->check_launch();
    });
}

int lane_b200_nccl_unique_id(void* id_out, size_t id_bytes) {
    return guard([&] { nccl_unique_id(id_out, id_bytes); });
}

int lane_b200_comm_init(lane_b200_ctx* c, int rank, int world, const void* id, size_t id_bytes) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        LANE_CUDA(cudaSetDevice(c->device));
        comm_init(c->comm, rank, world, id, id_bytes);
    });
}

int lane_b200_comm_destroy(lane_b200_ctx* c) {
    return guard([&] {
        if (!c) throw Error(LANE_ERR_CONFIG, "null context");
        comm_destroy(c->comm);
    });
}

int lane_b200_allreduce_grads(lane_b200_net* net) {
    return guard([&] {
        if (!net) throw Error(LANE_ERR_CONFIG, "null network");
        allreduce_grads(net->ctx->comm, net->grads, net->grads_count, net->ctx->stream);
    });
}

int lane_b200_nvls_supported(lane_b200_ctx* c, int* out) {
    return guard([&] {
        if (!c || !out) throw Error(LANE_ERR_CONFIG, "null argument");
        *out = nvls_supported(c->device) ? 1 : 0;
    });
}

// the arena plus one 256-byte barrier counter, multicast-bound
static size_t nvls_arena_bytes(const lane_b200_net* net) { return net->arena_bytes + 256; }

int lane_b200_nvls_create(lane_b200_net* net, int world, int* fd_out) {
    return guard([&] {
        if (!net || world < 1) throw Error(LANE_ERR_CONFIG, "nvls_create: bad arguments");
        if (net->nvls.mc || net->nvls.local) throw Error(LANE_ERR_CONFIG, "nvls_create: already created");
        LANE_CUDA(cudaSetDevice(net->ctx->device));
        nvls_create(net->nvls, net->ctx->device, world, nvls_arena_bytes(net));
        if (fd_out) *fd_out = nvls_export_fd(net->nvls);
    });
}

int lane_b200_nvls_attach(lane_b200_net* net, int rank, int world, int fd) {
    return guard([&] {
        if (!net || world < 1 || rank < 0 || rank >= world) throw Error(LANE_ERR_CONFIG, "nvls_attach: bad rank/world");
        LANE_CUDA(cudaSetDevice(net->ctx->device));
        if (rank != 0) {
            if (net->nvls.mc) throw Error(LANE_ERR_CONFIG, "nvls_attach: already attached");
            nvls_import(net->nvls, net->ctx->device, world, nvls_arena_bytes(net), fd);
        } else if ((!net->nvls.mc && !net->nvls.local) || net->nvls.world != world) {
            throw Error(LANE_ERR_CONFIG, "nvls_attach: rank 0 must nvls_create first (same world)");
        }
        nvls_add_device(net->nvls, rank);
    });
}

int lane_b200_nvls_mode(lane_b200_net* net, int* multicast) {
    return guard([&] {
        if (!net || !multicast) throw Error(LANE_ERR_CONFIG, "null argument");
        *multicast = !net->nvls.bound ? -1 : net->nvls.local ? 0 : 1;
    });
}

int lane_b200_nvls_bind(lane_b200_net* net) {
    return guard([&] {
        if (!net || !net->nvls.attached || net->nvls.bound) throw Error(LANE_ERR_CONFIG, "nvls_bind: not attached");
        auto* c = net->ctx;
        LANE_CUDA(cudaSetDevice(c->device));
        LANE_CUDA(cudaStreamSynchronize(c->stream));
        char* old = net->arena;
        char* base = nvls_bind(net->nvls);
        // move the arena (weights, velocities, activations) into the bound memory
        LANE_CUDA(cudaMemcpy(base, old, net->arena_bytes, cudaMemcpyDeviceToDevice));
        LANE_CUDA(cudaMemset(base + net->arena_bytes, 0, 256));  // barrier counter
        auto rebase = [&](auto*& p) {
            using T = std::remove_reference_t<decltype(*p)>;
            char* q = reinterpret_cast<char*>(p);
            if (q >= old && q < old + net->arena_bytes) p = reinterpret_cast<T*>(base + (q - old));
        };
        for (auto& Ly : net->layers)
            for (auto& b : Ly.buf) rebase(b);
        rebase(net->params);
        rebase(net->grads);
        rebase(net->target_stage);
        net->arena = base;
        net->mb_graph.reset();
        LANE_CUDA(cudaFree(old));
        LANE_CUDA(cudaDeviceSynchronize());
    });
}

}  // extern "C"
