// sgd_persistent.cuh -- fused online-SGD for the reference's one-hidden-layer
// topology (tanh FC -> softmax/CE), batch 1, as ONE persistent kernel.
//
// Reference per sample (network.cpp:164-170 -> :122-138, layers.hpp:28-61,
// layers.cpp:18-49, :71-87):
//   forward:  z0 = x W0 + b0, a = tanh(z0);  z1 = a W1 + b1, p = softmax(z1)
//   backward: d1 = p - t;  d0 = (1 - a^2) * (W1 d1)   (pre-update W1)
//   update:   W1 += -eta (a (x) d1); b1 += -eta d1; W0 += -eta (x (x) d0); b0 += -eta d0
//
// B200 design:
//  * The hidden neurons are partitioned across G co-resident CTAs (cooperative
//    launch).  CTA c owns columns [h0, h1) of W0 and the matching rows of W1;
//    both slices live in SHARED MEMORY for the whole sample stream (weights
//    never touch HBM between samples; up to ~29 MB across 148 SMs).
//  * Everything except the 10-wide logit reduction is CTA-local.  Each sample
//    needs exactly one cross-CTA exchange: every CTA publishes its C partial
//    logits as 64-bit {value, sample-tag} words (single-copy atomic, so the
//    tag doubles as the arrival flag -- no separate barrier), then every CTA
//    gathers all G*C words from L2 and reduces them in a fixed order, so all
//    CTAs hold bit-identical logits / probabilities / output deltas.
//  * The update of sample s is applied lazily while sample s+1 streams the
//    same smem weights through its forward dot products (one read-modify-write
//    pass over each weight per sample, the algorithmic minimum).  The update
//    arithmetic is the reference's exactly: w + (-eta * (delta * x)), three
//    separately rounded operations.
//  * The next sample's x/t rows are prefetched with cp.async into a triple
//    buffer (x(s-1) for the lazy update, x(s) for the forward, x(s+1) landing).
//  * tanh/exp/log are the bit-exact glibc restatements (lane_libm.cuh).  The
//    dot products are FMA trees (FAST numerics); STRICT numerics use the
//    layer-kernel path instead.
#pragma once

#include "common.cuh"

namespace lane_b200 {


struct SgdArgs {
    int I, H, C;
    int G;    // co-resident CTAs
    int npc;  // hidden neurons per CTA (max)
    int wpn;  // warps cooperating on one neuron's forward dot product
    const float* X;
    const float* T;
    const uint32_t* order;
    long long n, n_steps;
    float neg_eta;
    float *W0, *b0, *W1, *b1;
    unsigned long long* slots;  // [2][G][C] {value bits | tag << 32}
    // reference LayerState buffers after the last sample
    float *x0, *z0, *a0, *d0, *db0;  // hidden layer
    float *x1, *z1, *a1, *d1, *db1;  // output layer
    double* loss_sum;
    unsigned long long* correct;
    int* error;  // set to 1 when an exchange times out (bug guard, never hangs)
    unsigned long long* trace;  // debug: per-phase clock64 of CTA 0 for the first kTraceSamples
    int chunks;                 // grid/streamed: K chunks per column group (<= kGrChunks)
    int col4;                   // grid/streamed: 128-bit column quads (H % 4 == 0, npc % 4 == 0)
    int debug;                  // diagnostics only: bit 0 = skip the bulk weight pass (timing probe)
};

constexpr int kTraceSamples = 64, kTracePhases = 16;
#define SGD_TRACE(ph)                                                                     \
    do {                                                                                  \
        if (A.trace && (tid == 0 || tid == 32 * (kClWarps - 1)) && rank == 0 &&          \
            s < kTraceSamples)                                                            \
            A.trace[s * kTracePhases + (ph)] = clock64();                                 \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v));
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

// ===========================================================================
// Cluster variant (the B=1 flagship): the whole hidden layer lives in ONE
// thread-block cluster (<= 16 CTAs on one GPC); weights stay in shared memory
// for the whole sample stream; the per-sample exchange of partial logits goes
// through distributed shared memory with remote mbarrier arrivals.
//
// Warp specialisation per CTA:
//   warp 0 ("critical"): the serial chain of sample s --
//       wait partials(s) -> logits -> softmax -> d1(s) -> d0(s)
//       -> z(s+1) = y(s+1) + (-eta d0(s)) q(s+1) + b0(s+1) -> a(s+1) = tanh
//       -> W1 update(s) fused with partial logits(s+1) -> push to peers.
//   warps 1..NB ("bulk"): the O(I x npc) weight pass of sample s, which is
//       OFF the critical path:  W0 <- W0 + (-eta)(d0(s) (x) x(s))   (exact
//       reference rounding) fused with y(s+2) = x(s+2) . W0(s+1) and
//       q(s+2) = x(s+2) . x(s+1); plus the cp.async prefetch of x/t.
// The split uses  x(s+1).W0(s+1) = x(s+1).W0(s) + (-eta d0(s)) (x(s+1).x(s))
// (exact in real arithmetic; FAST numerics, checked against the oracle within
// the stated tolerance).  The weights themselves receive exactly the
// reference's update sequence.
// ===========================================================================

constexpr int kClBulkWarps = 16;
constexpr int kClWarps = 1 + kClBulkWarps;
constexpr int kClThreads = 32 * kClWarps;
constexpr int kClMaxC = 32;  // classes handled by the critical warp's lanes
constexpr int kBarDelta = 1, kBarPass = 2, kBarBulk = 3;  // named barriers (0 = __syncthreads)

struct ClSmem {
    int I, C, Ip, Cp, npc, wpn, CS;
    size_t w0s, w1s, xb, tb, b0s, abuf, zcur, d0, zl, pl, dl, gat, red, qred, mbar, total;
    __host__ __device__ ClSmem(int I_, int C_, int npc_, int wpn_, int CS_)
        : I(I_), C(C_), npc(npc_), wpn(wpn_), CS(CS_) {
        Ip = (I + 3) & ~3;
        Cp = (C + 3) & ~3;
        size_t o = 0;
        auto take = [&](size_t n) {
            size_t at = o;
            o += (n + 3) & ~size_t(3);
            return at;
        };
        w0s = take((size_t)npc * Ip);          // [j][i], rows zero-padded to Ip
        w1s = take((size_t)npc * C);           // [j][k]
        xb = take(4 * (size_t)Ip);             // x(s) ring, zero tails
        tb = take(4 * (size_t)Cp);             // t(s) ring
        b0s = take(npc);
        abuf = take(2 * (size_t)npc);          // a(s) by parity
        zcur = take(npc);
        d0 = take(2 * (size_t)npc);            // d0(s) by parity
        zl = take(Cp);
        pl = take(2 * (size_t)Cp);             // p(s) by parity
        dl = take(Cp);
        gat = take(2 * (size_t)CS * Cp);       // [parity][rank][k]
        red = take(2 * (size_t)npc * wpn);     // [parity][j][part]
        qred = take(2 * (size_t)wpn);          // [parity][part]
        mbar = take(4);                        // 2 x u64 mbarriers
        total = o * sizeof(float);
    }
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count) : "memory");
}
// local arrive that also raises the expected transaction bytes of the phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(addr), "r"(bytes)
                 : "memory");
}
// asynchronous remote store that completes 4 bytes of the remote mbarrier's
// transaction count on arrival: no fence, no separate arrive
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(
                     remote_addr),
                 "r"(__float_as_uint(v)), "r"(remote_mbar)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// cp.async of sample row k into an smem slot, issued by `nthreads` threads.
__device__ __forceinline__ void prefetch_row_k(const SgdArgs& A, long long k, float* xdst, float* tdst,
                                               int t, int nthreads) {
    const float* xs = A.X + k * A.I;
    const float* ts = A.T + k * A.C;
    if (((A.I & 3) == 0) && ((reinterpret_cast<uintptr_t>(xs) & 15) == 0)) {
        for (int q = t; q < (A.I >> 2); q += nthreads) cp_async16(xdst + 4 * q, xs + 4 * q);
    } else {
        for (int i = t; i < A.I; i += nthreads) cp_async4(xdst + i, xs + i);
    }
    for (int c = t; c < A.C; c += nthreads) cp_async4(tdst + c, ts + c);
}

__device__ __forceinline__ float4 sgd_apply4(float4 w, float neg_eta, float d, float4 x) {
    w.x = sgd_apply(w.x, neg_eta, d, x.x);
    w.y = sgd_apply(w.y, neg_eta, d, x.y);
    w.z = sgd_apply(w.z, neg_eta, d, x.z);
    w.w = sgd_apply(w.w, neg_eta, d, x.w);
    return w;
}
__device__ __forceinline__ float dot4(float4 a, float4 b, float acc) {
    acc = fmaf(a.x, b.x, acc);
    acc = fmaf(a.y, b.y, acc);
    acc = fmaf(a.z, b.z, acc);
    return fmaf(a.w, b.w, acc);
}

// CT: the class count as a compile-time constant (fully unrolled class loops),
// or 0 for a runtime C <= 32.
template <int CT>
__global__ void __launch_bounds__(kClThreads, 1) k_sgd_cluster(SgdArgs A) {
    extern __shared__ __align__(16) float sm[];
    const ClSmem L(A.I, A.C, A.npc, A.wpn, A.G);
    float* w0s = sm + L.w0s;
    float* w1s = sm + L.w1s;
    float* b0s = sm + L.b0s;
    float* abuf = sm + L.abuf;
    float* zcur = sm + L.zcur;
    float* d0b = sm + L.d0;
    float* zl = sm + L.zl;
    float* plb = sm + L.pl;
    float* dl = sm + L.dl;
    float* gat = sm + L.gat;
    float* red = sm + L.red;
    float* qred = sm + L.qred;
    const uint32_t mbar0 = smem_u32(sm + L.mbar);  // mbar[b] at mbar0 + 8*b

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, CS = A.G, Ip = L.Ip, Cp = L.Cp;
    const int C = CT > 0 ? CT : A.C;
    const int rank = (int)cluster_ctarank();
    const int h0 = min(H, rank * A.npc), h1 = min(H, h0 + A.npc), nloc = h1 - h0;
    const float neg_eta = A.neg_eta;
    const int wpn = A.wpn, nper = kClBulkWarps / wpn;
    const int n = (int)A.n_steps;
    float* const xb0 = sm + L.xb;
    float* const tb0 = sm + L.tb;
    auto xrow = [&](int s) { return xb0 + (s & 3) * Ip; };
    auto trow = [&](int s) { return tb0 + (s & 3) * Cp; };
    // The critical warp is the LAST warp: the warp arbiter favours the highest
    // warp id, so the serial chain wins issue slots over the bulk pass.
    const bool critical = warp == kClWarps - 1;

    // ---------------- prologue ----------------
    for (int e = tid; e < 4 * Ip; e += kClThreads) sm[L.xb + e] = 0.0f;  // zero tails
    for (int e = tid; e < nloc * Ip; e += kClThreads) {
        const int j = e / Ip, i = e - j * Ip;
        w0s[e] = i < I ? A.W0[(size_t)i * H + h0 + j] : 0.0f;
    }
    for (int e = tid; e < nloc * C; e += kClThreads) w1s[e] = A.W1[(size_t)h0 * C + e];
    for (int j = tid; j < nloc; j += kClThreads) b0s[j] = A.b0[h0 + j];
    const uint32_t xbytes = (uint32_t)(CS * Cp * sizeof(float));
    if (tid == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (n > 0) mbar_arrive_expect_tx(mbar0, xbytes);
        if (n > 1) mbar_arrive_expect_tx(mbar0 + 8, xbytes);
    }
    __syncthreads();
    for (int s = 0; s < 3 && s < n; ++s) {
        const long long k = A.order ? (long long)A.order[s] : s % A.n;
        prefetch_row_k(A, k, xrow(s), trow(s), tid, kClThreads);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // z(0) = x0.W0 -> red[0], y(1) = x1.W0 -> red[1], q(1) = x1.x0 (bulk warps)
    if (!critical) {
        const float4* x0 = reinterpret_cast<const float4*>(xrow(0));
        const float4* x1 = reinterpret_cast<const float4*>(xrow(1));
        const int Ip4 = Ip >> 2;
        for (int r = 0; r * nper < nloc; ++r) {
            const int jl = r * nper + warp / wpn, part = warp % wpn;
            if (jl >= nloc) continue;
            const int q0 = part * Ip4 / wpn, q1 = (part + 1) * Ip4 / wpn;
            const float4* wrow = reinterpret_cast<const float4*>(w0s + (size_t)jl * Ip);
            float a0 = 0.0f, a1 = 0.0f, aq = 0.0f;
            for (int q = q0 + lane; q < q1; q += 32) {
                const float4 w = wrow[q], u = x0[q], v = x1[q];
                a0 = dot4(u, w, a0);
                a1 = dot4(v, w, a1);
                if (jl == 0) aq = dot4(v, u, aq);
            }
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            aq = warp_sum(aq);
            if (lane == 0) {
                red[(size_t)jl * wpn + part] = a0;
                red[(size_t)(L.npc * wpn) + (size_t)jl * wpn + part] = a1;
                if (jl == 0) qred[wpn + part] = aq;
            }
        }
    }
    __syncthreads();
    const uint32_t gat_base = smem_u32(gat);
    // critical-warp registers: lane k owns class k, lane j owns neuron j (< 32)
    float b1k = 0.0f, Pk = 0.0f;
    if (critical) {
        if (lane < C) b1k = A.b1[lane];
        if (n > 0) {
            for (int j = lane; j < nloc; j += 32) {
                float z = red[(size_t)j * wpn];
                for (int p = 1; p < wpn; ++p) z += red[(size_t)j * wpn + p];
                z = sadd(z, b0s[j]);
                zcur[j] = z;
                abuf[j] = tanhf(z);
            }
            __syncwarp();
            if (lane < C)
                for (int j = 0; j < nloc; ++j) Pk = fmaf(abuf[j], w1s[(size_t)j * C + lane], Pk);
        }
    }
    cluster_sync_all();  // every CTA initialised (mbarriers, smem) before remote traffic
    if (critical && n > 0 && lane < Cp) {
        const uint32_t off = gat_base + (uint32_t)((rank * Cp + lane) * sizeof(float));
        for (int p = 0; p < CS; ++p) st_async_f32(mapa_shared(off, p), Pk, mapa_shared(mbar0, p));
    }
    if (!critical) {
        __threadfence_block();
        named_arrive(kBarPass, kClThreads);  // "pass(-1) done": y(1), q(1) ready
    }
    long long kpre = A.n > 0 ? 3 % A.n : 0;  // bulk: row of the next prefetch
    double loss_acc = 0.0;
    unsigned long long correct_acc = 0;
    const bool stats = rank == 0 && tid == 32 * (kClBulkWarps - 1);  // last bulk warp, lane 0
    if (stats && A.loss_sum) loss_acc = *A.loss_sum;

    // bulk warp geometry (loop-invariant): neuron slot, K part, float4 range
    const int jw = warp / wpn, part = warp % wpn, nrounds = (nloc + nper - 1) / nper;
    const int q0 = part * (Ip >> 2) / wpn, q1 = (part + 1) * (Ip >> 2) / wpn;

    // ---------------- the sample stream ----------------
    for (int s = 0; s < n; ++s) {
        const int par = s & 1;
        float* pl = plb + par * Cp;
        float* d0 = d0b + par * L.npc;
        if (critical) {
            const float* acur = abuf + par * L.npc;
            float* anxt = abuf + (par ^ 1) * L.npc;
            const uint32_t mb = mbar0 + 8 * par;
            SGD_TRACE(0);
            while (!mbar_try_wait(mb, (uint32_t)((s >> 1) & 1))) {
            }
            // re-arm for sample s+2 (peers cannot send s+2 before they hold
            // this CTA's partials of s+1, which are sent below)
            if (lane == 0 && s + 2 < n) mbar_arrive_expect_tx(mb, xbytes);
            SGD_TRACE(1);
            // -- logits, softmax, output deltas
            const float* tc = trow(s);
            float zk = -INFINITY, e = 0.0f, dk = 0.0f;
            if (lane < C) {
                const float* g = gat + (size_t)par * CS * Cp + lane;
                float v0 = 0.0f, v1 = 0.0f, v2 = 0.0f, v3 = 0.0f;
                int c = 0;
                for (; c + 4 <= CS; c += 4) {
                    v0 += g[(size_t)(c + 0) * Cp];
                    v1 += g[(size_t)(c + 1) * Cp];
                    v2 += g[(size_t)(c + 2) * Cp];
                    v3 += g[(size_t)(c + 3) * Cp];
                }
                for (; c < CS; ++c) v0 += g[(size_t)c * Cp];
                zk = sadd((v0 + v1) + (v2 + v3), b1k);
            }
            const float m = warp_max(zk);
            if (lane < C) e = expf(zk - m);
            const float sum = warp_sum(e);
            if (lane < C) {
                const float pk = __fdiv_rn(e, sum);
                dk = ssub(pk, tc[lane]);
                zl[lane] = zk;
                pl[lane] = pk;
                dl[lane] = dk;
            }
            __syncwarp();
            SGD_TRACE(2);
            // -- hidden deltas with W1(s) (sequential k, reference rounding)
            for (int j = lane; j < nloc; j += 32) {
                const float* wrow = w1s + (size_t)j * C;
                float acc = 0.0f;
                if constexpr (CT > 0) {
                    float wv[CT], dv[CT];
#pragma unroll
                    for (int k = 0; k < CT; ++k) {
                        wv[k] = wrow[k];
                        dv[k] = dl[k];
                    }
#pragma unroll
                    for (int k = 0; k < CT; ++k) acc = sadd(acc, smul(dv[k], wv[k]));
                } else {
                    for (int k = 0; k < C; ++k) acc = sadd(acc, smul(dl[k], wrow[k]));
                }
                d0[j] = tanh_grad(acur[j], acc);
            }
            __syncwarp();
            SGD_TRACE(3);
            named_sync(kBarPass, kClThreads);  // pass(s-1) done: y(s+1), q(s+1), t(s+1)
            SGD_TRACE(4);
            __threadfence_block();
            named_arrive(kBarDelta, kClThreads);  // release d0(s), p(s)
            if (s + 1 < n) {
                // -- z(s+1) = y(s+1) + (-eta d0(s)) q(s+1) + b0(s+1);  a(s+1) = tanh
                const int pn = par ^ 1;
                float qv = 0.0f;
                for (int p = 0; p < wpn; ++p) qv += qred[pn * wpn + p];
                for (int j = lane; j < nloc; j += 32) {
                    const float dj = d0[j];
                    const float b = sadd(b0s[j], smul(neg_eta, dj));
                    b0s[j] = b;
                    const float* ry = red + (size_t)pn * L.npc * wpn + (size_t)j * wpn;
                    float y = ry[0];
                    for (int p = 1; p < wpn; ++p) y += ry[p];
                    const float z = sadd(fmaf(neg_eta * dj, qv, y), b);
                    anxt[j] = tanhf(z);
                    zcur[j] = z;
                }
                __syncwarp();
                SGD_TRACE(5);
                // -- W1 update of sample s fused with the partial logits of s+1
                Pk = 0.0f;
                if (lane < C) {
                    float P1 = 0.0f;
                    int j = 0;
                    for (; j + 2 <= nloc; j += 2) {
                        float* wa = w1s + (size_t)j * C + lane;
                        float* wb = wa + C;
                        const float na = sgd_apply(*wa, neg_eta, dk, acur[j]);
                        const float nb = sgd_apply(*wb, neg_eta, dk, acur[j + 1]);
                        *wa = na;
                        *wb = nb;
                        Pk = fmaf(anxt[j], na, Pk);
                        P1 = fmaf(anxt[j + 1], nb, P1);
                    }
                    if (j < nloc) {
                        float* wa = w1s + (size_t)j * C + lane;
                        const float na = sgd_apply(*wa, neg_eta, dk, acur[j]);
                        *wa = na;
                        Pk = fmaf(anxt[j], na, Pk);
                    }
                    Pk += P1;
                    b1k = sadd(b1k, smul(neg_eta, dk));
                }
                SGD_TRACE(6);
                // -- push partial(s+1, k) to every peer (lane k sends its class)
                if (lane < Cp) {
                    const uint32_t off = gat_base + (uint32_t)(((pn * CS + rank) * Cp + lane) * sizeof(float));
                    const uint32_t mbn = mbar0 + 8 * pn;
                    for (int p = 0; p < CS; ++p) st_async_f32(mapa_shared(off, p), Pk, mapa_shared(mbn, p));
                }
                __syncwarp();
                SGD_TRACE(7);
            }
        } else {
            named_sync(kBarDelta, kClThreads);  // d0(s), p(s) visible
            SGD_TRACE(8);
            if (stats) {
                // loss / accuracy of sample s (network.cpp:165-168)
                const float* tc = trow(s);
                float loss = 0.0f;
                int bp = 0, btg = 0;
                for (int o = 0; o < C; ++o) {
                    if (tc[o] != 0.0f) {
                        const float q = pl[o] < 1e-12f ? 1e-12f : pl[o];
                        loss = ssub(loss, smul(tc[o], logf(q)));
                    }
                    if (pl[o] > pl[bp]) bp = o;
                    if (tc[o] > tc[btg]) btg = o;
                }
                loss_acc = __dadd_rn(loss_acc, (double)loss);
                correct_acc += bp == btg;
            }
            // prefetch x/t(s+3); make x(s+2) resident
            if (s + 3 < n) {
                const long long kk = A.order ? (long long)A.order[s + 3] : kpre;
                prefetch_row_k(A, kk, xrow(s + 3), trow(s + 3), tid, 32 * kClBulkWarps);
                if (++kpre == A.n) kpre = 0;
            }
            cp_async_commit();
            cp_async_wait<1>();
            named_sync(kBarBulk, 32 * kClBulkWarps);  // cp.async data visible to all bulk warps
            SGD_TRACE(9);
            if (A.debug & 1) {  // timing probe: critical chain alone
                __threadfence_block();
                named_arrive(kBarPass, kClThreads);
                continue;
            }
            // -- pass(s): W0 update of sample s fused with y(s+2), q(s+2);
            //    128-bit shared-memory traffic (4 weights per access)
            const float4* xs = reinterpret_cast<const float4*>(xrow(s));
            const float4* x1 = reinterpret_cast<const float4*>(xrow(s + 1));
            const float4* x2 = reinterpret_cast<const float4*>(xrow(s + 2));
            const bool do_y = s + 2 < n;
            for (int r = 0; r < nrounds; ++r) {
                const int jl = r * nper + jw;
                if (jl >= nloc) continue;
                float4* wrow = reinterpret_cast<float4*>(w0s + (size_t)jl * Ip);
                const float dj = d0[jl];
                if (do_y) {
                    float acc0 = 0.0f, acc1 = 0.0f, aq = 0.0f;
                    const bool qrow = jl == 0;
                    int q = q0 + lane;
                    for (; q + 32 < q1; q += 64) {
                        const float4 wa = sgd_apply4(wrow[q], neg_eta, dj, xs[q]);
                        const float4 wb = sgd_apply4(wrow[q + 32], neg_eta, dj, xs[q + 32]);
                        wrow[q] = wa;
                        wrow[q + 32] = wb;
                        const float4 ua = x2[q], ub = x2[q + 32];
                        acc0 = dot4(ua, wa, acc0);
                        acc1 = dot4(ub, wb, acc1);
                        if (qrow) aq = dot4(ua, x1[q], dot4(ub, x1[q + 32], aq));
                    }
                    if (q < q1) {
                        const float4 wa = sgd_apply4(wrow[q], neg_eta, dj, xs[q]);
                        wrow[q] = wa;
                        const float4 ua = x2[q];
                        acc0 = dot4(ua, wa, acc0);
                        if (qrow) aq = dot4(ua, x1[q], aq);
                    }
                    const float acc = warp_sum(acc0 + acc1);
                    if (qrow) aq = warp_sum(aq);
                    if (lane == 0) {
                        red[(size_t)par * L.npc * wpn + (size_t)jl * wpn + part] = acc;
                        if (qrow) qred[par * wpn + part] = aq;
                    }
                } else {
                    for (int q = q0 + lane; q < q1; q += 32) wrow[q] = sgd_apply4(wrow[q], neg_eta, dj, xs[q]);
                }
            }
            SGD_TRACE(10);
            __threadfence_block();
            named_arrive(kBarPass, kClThreads);
        }
    }
    if (critical && n > 0) named_sync(kBarPass, kClThreads);  // consume pass(n-1)'s arrival
    cp_async_wait<0>();
    __syncthreads();

    // ---------------- write back (W0 already final; W1/biases: last update) ----------------
    if (n > 0) {
        const int lp = (n - 1) & 1;
        const float* xl = xrow(n - 1);
        const float* al = abuf + lp * L.npc;
        const float* dlast = d0b + lp * L.npc;
        for (int e = tid; e < nloc * I; e += kClThreads) {
            const int j = e / I, i = e - j * I;
            A.W0[(size_t)i * H + h0 + j] = w0s[(size_t)j * Ip + i];
        }
        for (int e = tid; e < nloc * C; e += kClThreads) {
            const int j = e / C, k = e - j * C;
            A.W1[(size_t)h0 * C + e] = sgd_apply(w1s[e], neg_eta, dl[k], al[j]);
        }
        for (int j = tid; j < nloc; j += kClThreads) {
            const float db = smul(neg_eta, dlast[j]);
            A.b0[h0 + j] = sadd(b0s[j], db);
            A.z0[h0 + j] = zcur[j];
            A.a0[h0 + j] = al[j];
            A.d0[h0 + j] = dlast[j];
            A.db0[h0 + j] = db;
            A.x1[h0 + j] = al[j];
        }
        if (critical && rank == 0 && lane < C) {
            const float db = smul(neg_eta, dl[lane]);
            A.b1[lane] = sadd(b1k, db);
            A.z1[lane] = zl[lane];
            A.a1[lane] = plb[lp * Cp + lane];
            A.d1[lane] = dl[lane];
            A.db1[lane] = db;
        }
        if (rank == 0)
            for (int i = tid; i < I; i += kClThreads) A.x0[i] = xl[i];
        if (stats) {
            if (A.loss_sum) *A.loss_sum = loss_acc;
            if (A.correct) *A.correct += correct_acc;
        }
    }
    cluster_sync_all();  // no CTA exits while a peer may still address its shared memory
}

// ===========================================================================
// Grid variant (large widths, e.g. 340-16384-10 and the paper's 340-100000-10):
// the same warp specialisation as k_sgd_cluster, over ALL SMs (cooperative
// launch, one CTA per SM).  The per-sample exchange of partial logits goes
// through L2 as 64-bit {value, sample tag} words (single-copy atomic, the tag
// doubles as the arrival flag).  W0 is either resident in shared memory
// (W0_SMEM, slices up to ~200 KB per SM) or streamed from HBM every sample in
// its native row-major layout with coalesced column access (the paper shape:
// 8 B per weight per sample, the algorithmic minimum -- HBM-bound).
// ===========================================================================

constexpr int kGrChunks = 32;  // max K chunks per column group in the streamed pass

struct GrSmem {
    int I, C, Ip, Cp, npc, G;
    bool w0_smem;
    size_t w0s, w1s, xb, tb, b0s, abuf, zcur, d0, zl, pl, dl, gat, red, qred, total;
    __host__ __device__ GrSmem(int I_, int C_, int npc_, int G_, bool w0_smem_, int chunks = 1)
        : I(I_), C(C_), npc(npc_), G(G_), w0_smem(w0_smem_) {
        Ip = (I + 3) & ~3;
        Cp = (C + 3) & ~3;
        size_t o = 0;
        auto take = [&](size_t n) {
            size_t at = o;
            o += (n + 3) & ~size_t(3);
            return at;
        };
        w0s = take(w0_smem ? (size_t)npc * Ip : 0);
        w1s = take((size_t)npc * C);
        xb = take(4 * (size_t)Ip);
        tb = take(4 * (size_t)Cp);
        b0s = take(npc);
        abuf = take(2 * (size_t)npc);
        zcur = take(npc);
        d0 = take(2 * (size_t)npc);
        zl = take(Cp);
        pl = take(2 * (size_t)Cp);
        dl = take(Cp);
        gat = take((size_t)G * Cp);
        red = take(2 * (size_t)npc * (w0_smem ? 1 : chunks));  // [parity][j][chunk]
        qred = take(2 * 4);
        total = o * sizeof(float);
    }
};

template <int CT, bool W0_SMEM>
__global__ void __launch_bounds__(kClThreads, 1) k_sgd_grid(SgdArgs A) {
    extern __shared__ __align__(16) float sm[];
    const GrSmem L(A.I, A.C, A.npc, A.G, W0_SMEM, A.chunks);
    float* w0s = sm + L.w0s;
    float* w1s = sm + L.w1s;
    float* b0s = sm + L.b0s;
    float* abuf = sm + L.abuf;
    float* zcur = sm + L.zcur;
    float* d0b = sm + L.d0;
    float* zl = sm + L.zl;
    float* plb = sm + L.pl;
    float* dl = sm + L.dl;
    float* gat = sm + L.gat;
    float* red = sm + L.red;
    float* qred = sm + L.qred;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, G = A.G, Ip = L.Ip, Cp = L.Cp;
    const int C = CT > 0 ? CT : A.C;
    const int cta = blockIdx.x;
    const int h0 = min(H, cta * A.npc), h1 = min(H, h0 + A.npc), nloc = h1 - h0;
    const float neg_eta = A.neg_eta;
    const int n = (int)A.n_steps;
    const int npc = L.npc;
    float* const xb0 = sm + L.xb;
    float* const tb0 = sm + L.tb;
    auto xrow = [&](int s) { return xb0 + (s & 3) * Ip; };
    auto trow = [&](int s) { return tb0 + (s & 3) * Cp; };
    const bool critical = warp == kClWarps - 1;
    constexpr int NB = 32 * kClBulkWarps;  // bulk threads
    // reductions per neuron: smem mode -> 1 (a warp owns a whole row);
    // streamed mode -> kGrChunks K-chunks per column
    const int NR = W0_SMEM ? 1 : A.chunks;

    // ---------------- prologue ----------------
    for (int e = tid; e < 4 * Ip; e += kClThreads) xb0[e] = 0.0f;
    if constexpr (W0_SMEM) {
        for (int e = tid; e < nloc * Ip; e += kClThreads) {
            const int j = e / Ip, i = e - j * Ip;
            w0s[e] = i < I ? A.W0[(size_t)i * H + h0 + j] : 0.0f;
        }
    }
    for (int e = tid; e < nloc * C; e += kClThreads) w1s[e] = A.W1[(size_t)h0 * C + e];
    for (int j = tid; j < nloc; j += kClThreads) b0s[j] = A.b0[h0 + j];
    __syncthreads();
    for (int s = 0; s < 3 && s < n; ++s) {
        const long long k = A.order ? (long long)A.order[s] : s % A.n;
        prefetch_row_k(A, k, xrow(s), trow(s), tid, kClThreads);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();

    // The bulk pass.  mode 0 (prologue): z(0) -> red[0], y(1) -> red[1], q(1);
    // mode 1 (sample s): W0 update of s, y(s+2) -> red[par], q(s+2) -> qred[par].
    auto bulk_pass = [&](int mode, int s) {
        const float* xs = mode ? xrow(s) : xrow(0);
        const float* x1 = mode ? xrow(s + 1) : xrow(1);
        const float* x2 = mode ? xrow(s + 2) : xrow(1);
        const bool do_y = mode ? (s + 2 < n) : true;
        const int py = mode ? (s & 1) : 1;
        const float* d0 = d0b + (s & 1) * npc;
        // q = x2 . x1 (prologue: x1 . x0), one warp
        if (warp == kClBulkWarps - 1 && do_y) {
            const float* qa = mode ? x1 : xrow(0);
            float aq = 0.0f;
            for (int i = lane; i < I; i += 32) aq = fmaf(x2[i], qa[i], aq);
            aq = warp_sum(aq);
            if (lane == 0) qred[py * 4] = aq;
        }
        if constexpr (W0_SMEM) {
            const int Ip4 = Ip >> 2;
            for (int jl = warp; jl < nloc; jl += kClBulkWarps) {
                float4* wrow = reinterpret_cast<float4*>(w0s + (size_t)jl * Ip);
                const float4* xs4 = reinterpret_cast<const float4*>(xs);
                const float4* x24 = reinterpret_cast<const float4*>(x2);
                const float4* x04 = reinterpret_cast<const float4*>(xrow(0));
                float acc0 = 0.0f, acc1 = 0.0f;
                if (mode == 0) {
                    for (int q = lane; q < Ip4; q += 32) {
                        const float4 w = wrow[q];
                        acc0 = dot4(x04[q], w, acc0);
                        acc1 = dot4(x24[q], w, acc1);
                    }
                    acc0 = warp_sum(acc0);
                    acc1 = warp_sum(acc1);
                    if (lane == 0) {
                        red[(size_t)jl * NR] = acc0;
                        red[(size_t)npc * NR + (size_t)jl * NR] = acc1;
                    }
                } else if (do_y) {
                    const float dj = d0[jl];
                    for (int q = lane; q < Ip4; q += 32) {
                        const float4 w = sgd_apply4(wrow[q], neg_eta, dj, xs4[q]);
                        wrow[q] = w;
                        acc0 = dot4(x24[q], w, acc0);
                    }
                    acc0 = warp_sum(acc0);
                    if (lane == 0) red[(size_t)py * npc * NR + (size_t)jl * NR] = acc0;
                } else {
                    const float dj = d0[jl];
                    for (int q = lane; q < Ip4; q += 32) wrow[q] = sgd_apply4(wrow[q], neg_eta, dj, xs4[q]);
                }
            }
        } else if (A.col4) {
            // streamed, 128-bit: items (chunk c, column quad jq); consecutive
            // threads -> consecutive 16-byte segments of one W0 row (coalesced);
            // 8 rows x 16 B in flight per thread
            const int quads = nloc >> 2, nch = A.chunks;
            const int items = quads * nch;
            for (int it = tid; it < items; it += NB) {
                const int c = it / quads, jq = it - c * quads;
                const int i0 = c * I / nch, i1 = (c + 1) * I / nch;
                float4* col = reinterpret_cast<float4*>(A.W0 + (size_t)(h0 + 4 * jq));
                const size_t H4 = (size_t)H >> 2;
                float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
                if (mode == 0) {
                    const float* x0 = xrow(0);
                    for (int i = i0; i < i1; ++i) {
                        const float4 w = __ldcg(col + (size_t)i * H4);
                        a0.x = fmaf(x0[i], w.x, a0.x); a0.y = fmaf(x0[i], w.y, a0.y);
                        a0.z = fmaf(x0[i], w.z, a0.z); a0.w = fmaf(x0[i], w.w, a0.w);
                        a1.x = fmaf(x2[i], w.x, a1.x); a1.y = fmaf(x2[i], w.y, a1.y);
                        a1.z = fmaf(x2[i], w.z, a1.z); a1.w = fmaf(x2[i], w.w, a1.w);
                    }
                    float* r0 = red + (size_t)(4 * jq) * NR + c;
                    float* r1 = red + (size_t)npc * NR + (size_t)(4 * jq) * NR + c;
                    r0[0] = a0.x; r0[NR] = a0.y; r0[2 * NR] = a0.z; r0[3 * NR] = a0.w;
                    r1[0] = a1.x; r1[NR] = a1.y; r1[2 * NR] = a1.z; r1[3 * NR] = a1.w;
                } else {
                    const float4 dq = *reinterpret_cast<const float4*>(d0 + 4 * jq);
                    int i = i0;
                    for (; i + 8 <= i1; i += 8) {
                        float4 w[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) w[u] = __ldcg(col + (size_t)(i + u) * H4);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const float xv = xs[i + u], yv = x2[i + u];
                            w[u].x = sgd_apply(w[u].x, neg_eta, dq.x, xv);
                            w[u].y = sgd_apply(w[u].y, neg_eta, dq.y, xv);
                            w[u].z = sgd_apply(w[u].z, neg_eta, dq.z, xv);
                            w[u].w = sgd_apply(w[u].w, neg_eta, dq.w, xv);
                            __stcg(col + (size_t)(i + u) * H4, w[u]);
                            a0.x = fmaf(yv, w[u].x, a0.x); a0.y = fmaf(yv, w[u].y, a0.y);
                            a0.z = fmaf(yv, w[u].z, a0.z); a0.w = fmaf(yv, w[u].w, a0.w);
                        }
                    }
                    for (; i < i1; ++i) {
                        float4 w = __ldcg(col + (size_t)i * H4);
                        const float xv = xs[i], yv = x2[i];
                        w.x = sgd_apply(w.x, neg_eta, dq.x, xv);
                        w.y = sgd_apply(w.y, neg_eta, dq.y, xv);
                        w.z = sgd_apply(w.z, neg_eta, dq.z, xv);
                        w.w = sgd_apply(w.w, neg_eta, dq.w, xv);
                        __stcg(col + (size_t)i * H4, w);
                        a0.x = fmaf(yv, w.x, a0.x); a0.y = fmaf(yv, w.y, a0.y);
                        a0.z = fmaf(yv, w.z, a0.z); a0.w = fmaf(yv, w.w, a0.w);
                    }
                    if (do_y) {
                        float* r0 = red + (size_t)py * npc * NR + (size_t)(4 * jq) * NR + c;
                        r0[0] = a0.x; r0[NR] = a0.y; r0[2 * NR] = a0.z; r0[3 * NR] = a0.w;
                    }
                }
            }
        } else {
            // streamed, scalar (H % 4 != 0): items (chunk c, column j)
            const int nch = A.chunks;
            const int items = nloc * nch;
            for (int it = tid; it < items; it += NB) {
                const int c = it / nloc, jl = it - c * nloc;
                const int i0 = c * I / nch, i1 = (c + 1) * I / nch;
                float* col = A.W0 + (size_t)(h0 + jl);
                float acc0 = 0.0f, acc1 = 0.0f;
                if (mode == 0) {
                    const float* x0 = xrow(0);
                    for (int i = i0; i < i1; ++i) {
                        const float w = __ldcg(col + (size_t)i * H);
                        acc0 = fmaf(x0[i], w, acc0);
                        acc1 = fmaf(x2[i], w, acc1);
                    }
                    red[(size_t)jl * NR + c] = acc0;
                    red[(size_t)npc * NR + (size_t)jl * NR + c] = acc1;
                } else {
                    const float dj = d0[jl];
                    int i = i0;
                    for (; i + 8 <= i1; i += 8) {
                        float w[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) w[u] = __ldcg(col + (size_t)(i + u) * H);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            w[u] = sgd_apply(w[u], neg_eta, dj, xs[i + u]);
                            __stcg(col + (size_t)(i + u) * H, w[u]);
                            acc0 = fmaf(x2[i + u], w[u], acc0);
                        }
                    }
                    for (; i < i1; ++i) {
                        const float w = sgd_apply(__ldcg(col + (size_t)i * H), neg_eta, dj, xs[i]);
                        __stcg(col + (size_t)i * H, w);
                        acc0 = fmaf(x2[i], w, acc0);
                    }
                    if (do_y) red[(size_t)py * npc * NR + (size_t)jl * NR + c] = acc0;
                }
            }
        }
    };

    if (!critical) bulk_pass(0, 0);
    __syncthreads();
    float b1k = 0.0f, Pk = 0.0f;
    if (critical) {
        if (lane < C) b1k = A.b1[lane];
        if (n > 0) {
            for (int j = lane; j < nloc; j += 32) {
                float z = red[(size_t)j * NR];
                for (int p = 1; p < NR; ++p) z += red[(size_t)j * NR + p];
                z = sadd(z, b0s[j]);
                zcur[j] = z;
                abuf[j] = tanhf(z);
            }
            __syncwarp();
            if (lane < C) {
                float P0 = 0.0f, P1 = 0.0f;
                int j = 0;
                for (; j + 2 <= nloc; j += 2) {
                    P0 = fmaf(abuf[j], w1s[(size_t)j * C + lane], P0);
                    P1 = fmaf(abuf[j + 1], w1s[(size_t)(j + 1) * C + lane], P1);
                }
                if (j < nloc) P0 = fmaf(abuf[j], w1s[(size_t)j * C + lane], P0);
                Pk = P0 + P1;
                st_relaxed_u64(A.slots + (size_t)cta * C + lane,
                               (1ull << 32) | __float_as_uint(Pk));
            }
        }
    } else {
        __threadfence_block();
        named_arrive(kBarPass, kClThreads);
    }
    long long kpre = A.n > 0 ? 3 % A.n : 0;
    double loss_acc = 0.0;
    unsigned long long correct_acc = 0;
    const bool stats = cta == 0 && tid == 32 * (kClBulkWarps - 1);
    if (stats && A.loss_sum) loss_acc = *A.loss_sum;
    const int GC = G * C;

    for (int s = 0; s < n; ++s) {
        const int par = s & 1;
        float* pl = plb + par * Cp;
        float* d0 = d0b + par * npc;
        if (critical) {
            const float* acur = abuf + par * npc;
            float* anxt = abuf + (par ^ 1) * npc;
            // -- gather every CTA's partial logits of sample s from L2
            const uint32_t tag = (uint32_t)(s + 1);
            const unsigned long long* slot = A.slots + (size_t)par * GC;
            const unsigned long long t0 = globaltimer_ns();
            for (int base = lane; base < GC; base += 32 * 8) {
                unsigned long long v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = base + 32 * u;
                    v[u] = e < GC ? ld_relaxed_u64(slot + e) : ((unsigned long long)tag << 32);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = base + 32 * u;
                    if (e < GC) {
                        while ((uint32_t)(v[u] >> 32) != tag) {
                            if (globaltimer_ns() - t0 > 5000000000ull) {  // a bug, not a wait
                                atomicExch(A.error, 1);
                                __trap();
                            }
                            v[u] = ld_relaxed_u64(slot + e);
                        }
                        const int c = e / C, k = e - c * C;
                        gat[(size_t)c * Cp + k] = __uint_as_float((uint32_t)v[u]);
                    }
                }
            }
            __syncwarp();
            const float* tc = trow(s);
            float zk = -INFINITY, e = 0.0f, dk = 0.0f;
            if (lane < C) {
                const float* g = gat + lane;
                float v0 = 0.0f, v1 = 0.0f, v2 = 0.0f, v3 = 0.0f;
                int c = 0;
                for (; c + 4 <= G; c += 4) {
                    v0 += g[(size_t)(c + 0) * Cp];
                    v1 += g[(size_t)(c + 1) * Cp];
                    v2 += g[(size_t)(c + 2) * Cp];
                    v3 += g[(size_t)(c + 3) * Cp];
                }
                for (; c < G; ++c) v0 += g[(size_t)c * Cp];
                zk = sadd((v0 + v1) + (v2 + v3), b1k);
            }
            const float m = warp_max(zk);
            if (lane < C) e = expf(zk - m);
            const float sum = warp_sum(e);
            if (lane < C) {
                const float pk = __fdiv_rn(e, sum);
                dk = ssub(pk, tc[lane]);
                zl[lane] = zk;
                pl[lane] = pk;
                dl[lane] = dk;
            }
            __syncwarp();
            // -- hidden deltas with W1(s)
            for (int j = lane; j < nloc; j += 32) {
                const float* wrow = w1s + (size_t)j * C;
                float acc = 0.0f;
                if constexpr (CT > 0) {
                    float wv[CT], dv[CT];
#pragma unroll
                    for (int k = 0; k < CT; ++k) {
                        wv[k] = wrow[k];
                        dv[k] = dl[k];
                    }
#pragma unroll
                    for (int k = 0; k < CT; ++k) acc = sadd(acc, smul(dv[k], wv[k]));
                } else {
                    for (int k = 0; k < C; ++k) acc = sadd(acc, smul(dl[k], wrow[k]));
                }
                d0[j] = tanh_grad(acur[j], acc);
            }
            __syncwarp();
            named_sync(kBarPass, kClThreads);
            __threadfence_block();
            named_arrive(kBarDelta, kClThreads);
            if (s + 1 < n) {
                const int pn = par ^ 1;
                const float qv = qred[pn * 4];
                for (int j = lane; j < nloc; j += 32) {
                    const float dj = d0[j];
                    const float b = sadd(b0s[j], smul(neg_eta, dj));
                    b0s[j] = b;
                    const float* ry = red + (size_t)pn * npc * NR + (size_t)j * NR;
                    float y = ry[0];
                    for (int p = 1; p < NR; ++p) y += ry[p];
                    const float z = sadd(fmaf(neg_eta * dj, qv, y), b);
                    anxt[j] = tanhf(z);
                    zcur[j] = z;
                }
                __syncwarp();
                if (lane < C) {
                    float P0 = 0.0f, P1 = 0.0f;
                    int j = 0;
                    for (; j + 2 <= nloc; j += 2) {
                        float* wa = w1s + (size_t)j * C + lane;
                        float* wb = wa + C;
                        const float na = sgd_apply(*wa, neg_eta, dk, acur[j]);
                        const float nb = sgd_apply(*wb, neg_eta, dk, acur[j + 1]);
                        *wa = na;
                        *wb = nb;
                        P0 = fmaf(anxt[j], na, P0);
                        P1 = fmaf(anxt[j + 1], nb, P1);
                    }
                    if (j < nloc) {
                        float* wa = w1s + (size_t)j * C + lane;
                        const float na = sgd_apply(*wa, neg_eta, dk, acur[j]);
                        *wa = na;
                        P0 = fmaf(anxt[j], na, P0);
                    }
                    Pk = P0 + P1;
                    b1k = sadd(b1k, smul(neg_eta, dk));
                    st_relaxed_u64(A.slots + (size_t)pn * GC + (size_t)cta * C + lane,
                                   ((unsigned long long)(s + 2) << 32) | __float_as_uint(Pk));
                }
                __syncwarp();
            }
        } else {
            named_sync(kBarDelta, kClThreads);
            if (stats) {
                const float* tc = trow(s);
                float loss = 0.0f;
                int bp = 0, btg = 0;
                for (int o = 0; o < C; ++o) {
                    if (tc[o] != 0.0f) {
                        const float q = pl[o] < 1e-12f ? 1e-12f : pl[o];
                        loss = ssub(loss, smul(tc[o], logf(q)));
                    }
                    if (pl[o] > pl[bp]) bp = o;
                    if (tc[o] > tc[btg]) btg = o;
                }
                loss_acc = __dadd_rn(loss_acc, (double)loss);
                correct_acc += bp == btg;
            }
            if (s + 3 < n) {
                const long long kk = A.order ? (long long)A.order[s + 3] : kpre;
                prefetch_row_k(A, kk, xrow(s + 3), trow(s + 3), tid, NB);
                if (++kpre == A.n) kpre = 0;
            }
            cp_async_commit();
            cp_async_wait<1>();
            named_sync(kBarBulk, NB);
            bulk_pass(1, s);
            __threadfence_block();
            named_arrive(kBarPass, kClThreads);
        }
    }
    if (critical && n > 0) named_sync(kBarPass, kClThreads);
    cp_async_wait<0>();
    __syncthreads();

    if (n > 0) {
        const int lp = (n - 1) & 1;
        const float* xl = xrow(n - 1);
        const float* al = abuf + lp * npc;
        const float* dlast = d0b + lp * npc;
        if constexpr (W0_SMEM) {
            for (int e = tid; e < nloc * I; e += kClThreads) {
                const int j = e / I, i = e - j * I;
                A.W0[(size_t)i * H + h0 + j] = w0s[(size_t)j * Ip + i];
            }
        }
        for (int e = tid; e < nloc * C; e += kClThreads) {
            const int j = e / C, k = e - j * C;
            A.W1[(size_t)h0 * C + e] = sgd_apply(w1s[e], neg_eta, dl[k], al[j]);
        }
        for (int j = tid; j < nloc; j += kClThreads) {
            const float db = smul(neg_eta, dlast[j]);
            A.b0[h0 + j] = sadd(b0s[j], db);
            A.z0[h0 + j] = zcur[j];
            A.a0[h0 + j] = al[j];
            A.d0[h0 + j] = dlast[j];
            A.db0[h0 + j] = db;
            A.x1[h0 + j] = al[j];
        }
        if (critical && cta == 0 && lane < C) {
            const float db = smul(neg_eta, dl[lane]);
            A.b1[lane] = sadd(b1k, db);
            A.z1[lane] = zl[lane];
            A.a1[lane] = plb[lp * Cp + lane];
            A.d1[lane] = dl[lane];
            A.db1[lane] = db;
        }
        if (cta == 0)
            for (int i = tid; i < I; i += kClThreads) A.x0[i] = xl[i];
        if (stats) {
            if (A.loss_sum) *A.loss_sum = loss_acc;
            if (A.correct) *A.correct += correct_acc;
        }
    }
}

}  // namespace lane_b200
