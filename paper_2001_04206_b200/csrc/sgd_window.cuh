// sgd_window.cuh -- online SGD (batch 1) for the one-hidden-layer topology
// with the O(I x H) first-layer work taken OFF the per-sample dependency chain.
//
// Reference per sample (network.cpp:164-170 -> :122-138, layers.hpp:28-61,
// layers.cpp:18-49, :71-87):
//   forward:  z0 = x W0 + b0, a = tanh(z0);  z1 = a W1 + b1, p = softmax(z1)
//   backward: d1 = p - t;  d0 = (1 - a^2) * (W1 d1)   (pre-update W1)
//   update:   W1 += -eta (a (x) d1); b1 += -eta d1; W0 += -eta (x (x) d0); b0 += -eta d0
//
// Delayed-base identity (exact in real arithmetic).  With W0(s) the weights
// before sample s and any earlier base sample B <= s,
//   x(s).W0(s) = x(s).W0(B) + sum_{B<=r<s} (-eta x(s).x(r)) d0(r).
// Samples are grouped in blocks of S.  For a sample in block b the base is the
// end of block b-D, so
//   z0(s) = Y(s) + sum_{r in window(s)} c(s, s-r) d0(r) + b0(s),
//   Y(s)  = x(s).W0(after block b-D),  c(s, d) = -eta x(s).x(s-d)  (banded Gram).
// Only the H-wide chain (tanh, the H x C output layer, softmax, d1, d0) stays
// serial; everything O(I x H) is batched per block and runs D-1 blocks ahead.
//
// Roles (one cooperative launch, 1 + P CTAs, one per SM):
//  * CTA 0, the chain CTA:
//     - critical warp (highest id, favoured by the warp arbiter): the serial
//       chain of every sample; W1 (H x C) lives in its registers, lane l owns
//       hidden units [JPL*l, JPL*l+JPL); one transpose-reduce of the partial
//       logits; exact reference rounding for the W1/b1/b0 updates.
//     - helper warps: apply every new d0(r) to the pending z rows of the
//       window (row s is owned by helper s mod NH, so each row has one
//       writer); the owner of row s+2 signals it ready right after d0(s).
//     - loader warp: stages Y(b), the targets and c(s,1) of block b in shared
//       memory once the producers have published Y(b).
//     - publisher warp: copies each finished block's d0 rows to L2 for the
//       producers (release counter) and accumulates loss/accuracy off the
//       chain, in sample order.
//  * CTAs 1..P, the producers: CTA p owns W0 columns [4p, 4p+4) in registers
//    for the whole stream.  Per block k: acquire d0 of block k, apply the S
//    per-sample updates with the reference's exact rounding
//    (w + (-eta * (d0 * x)), sample by sample), then compute Y(k+D) from the
//    updated weights and release it.  The weights never leave the chip until
//    the final write-back.
// c(s,d) comes from a banded-Gram pre-pass (k_gram_band) over the same stream.
//
// Numerics: FAST (the forward dot products are reassociated); the weights
// receive exactly the reference's per-sample update sequence given d0.
#pragma once

#include "common.cuh"
#include "sgd_persistent.cuh"

namespace lane_b200 {

constexpr int kWinS = 16;                    // samples per block
constexpr int kWinHelpers = 8;               // helper warps
constexpr int kWinWarps = kWinHelpers + 3;   // + publisher, loader, critical
constexpr int kWinThreads = 32 * kWinWarps;  // 352
constexpr int kWinPub = kWinHelpers, kWinLoad = kWinHelpers + 1, kWinCrit = kWinHelpers + 2;
constexpr int kWinMaxD = 6;
constexpr int kWinRing = 16;                 // d0-ready / row-ready mbarrier rings
constexpr int kWinBlkRing = 8;               // block-done mbarrier ring (> D)
constexpr int kWinMaxNR = 4;                 // producer: W0 rows per thread (I <= 4 * 352)
constexpr int kWinCP = 16;                   // classes padded for the transpose-reduce
constexpr int kWinMaxMine = (kWinMaxD * kWinS + kWinHelpers - 1) / kWinHelpers;

struct WinArgs {
    int I, H, C, D, P, QW;
    const float* X;
    const float* T;
    const uint32_t* order;  // stream order (offset to this launch) or null
    long long n;            // dataset rows
    long long n_steps;      // samples in this launch
    long long base;         // first stream position (no order: row = (base + s) % n)
    float neg_eta;
    float *W0, *b0, *W1, *b1;
    float* coef;        // [n_steps][QW]: c(s, d) at [s][d-1]
    float* yring;       // [D+1][S][H]
    float* dring;       // [D+1][S][H]
    unsigned* ycnt;     // [D+1] monotonic producer arrivals per Y slot
    unsigned* dcnt;     // published d0 blocks
    float *x0, *z0, *a0, *d0, *db0;
    float *x1, *z1, *a1, *d1, *db1;
    double* loss_sum;
    unsigned long long* correct;
    int* error;
    unsigned long long* trace;
};

struct WinSmem {
    int HP, R, Rd;
    size_t zacc, ystage, tstage, c1stage, d0ring, pring, red, d0s, mbar, total;
    __host__ __device__ WinSmem(int HP_, int D) : HP(HP_) {
        R = D * kWinS;
        Rd = (D + 1) * kWinS;
        size_t o = 0;
        auto take = [&](size_t nf) {
            size_t at = o;
            o += (nf + 3) & ~size_t(3);
            return at;
        };
        zacc = take((size_t)R * HP);
        ystage = take(2 * (size_t)kWinS * HP);
        tstage = take(2 * kWinS * kWinCP);
        c1stage = take(2 * kWinS);
        d0ring = take((size_t)Rd * HP);
        pring = take((size_t)Rd * kWinCP);
        red = take(kWinWarps * 64);
        d0s = take(kWinS * 4);
        mbar = take(2 * (2 * kWinRing + 4 + kWinBlkRing));
        total = o * sizeof(float);
    }
};

// mbarrier indices (u64 slots)
constexpr int kMbD0 = 0, kMbRow = kWinRing, kMbYFull = 2 * kWinRing, kMbYFree = 2 * kWinRing + 2,
              kMbBlk = 2 * kWinRing + 4;

__device__ __forceinline__ void mbar_arrive_cta(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ bool mbar_test_cta(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
// a 5 s stall is a protocol bug: trap rather than hang the GPU
__device__ __noinline__ void mbar_wait_slow(uint32_t a, uint32_t parity, int* err) {
    const unsigned long long t0 = globaltimer_ns();
    while (!mbar_test_cta(a, parity)) {
        if (globaltimer_ns() - t0 > 5000000000ull) {
            atomicExch(err, 3);
            __trap();
        }
    }
}
__device__ __forceinline__ void mbar_wait_cta(uint32_t a, uint32_t parity, int* err) {
    if (!mbar_test_cta(a, parity)) mbar_wait_slow(a, parity, err);
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// spin on a monotonic L2 counter; a 5 s stall is a bug, never a wait
__device__ __forceinline__ void spin_geq(const unsigned* p, unsigned target, int* err) {
    if (ld_acquire_u32(p) >= target) return;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_u32(p) < target) {
        if (globaltimer_ns() - t0 > 5000000000ull) {
            atomicExch(err, 2);
            __trap();
        }
    }
}

__device__ __forceinline__ long long win_row(const WinArgs& A, long long s) {
    return A.order ? (long long)A.order[s] : (A.base + s) % A.n;
}

// Transpose-reduce of N per-lane values over the lanes selected by the
// butterfly offsets 16, 8, ..., OMIN: after the step with offset o each lane
// keeps half of its values (the half selected by its lane bit o) summed with
// the partner's copy.  Fixed tree: deterministic.
template <int N>
__device__ __forceinline__ void xpose_step(float* v, int lane, int o) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
        const float send = hi ? v[q] : v[q + N / 2];
        const float keep = hi ? v[q + N / 2] : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
}

// ---------------------------------------------------------------------------
// Banded Gram pre-pass: coef[s][d-1] = -eta * (x(s) . x(s-d)), d = 1..QW
// (0 when s-d < 0).  One CTA per 32 stream positions; K streamed through
// shared memory in 32-float chunks; thread (s, d-group) accumulates QW/8 dots.
// ---------------------------------------------------------------------------
constexpr int kGramTS = 32, kGramKC = 32, kGramMaxQW = 96;

__global__ void __launch_bounds__(256) k_gram_band(WinArgs A) {
    __shared__ float xs[kGramTS + kGramMaxQW][kGramKC + 1];
    __shared__ long long rows[kGramTS + kGramMaxQW];
    const int QW = A.QW, I = A.I;
    const long long s0 = (long long)blockIdx.x * kGramTS;
    const int NRW = kGramTS + QW;  // rows s0-QW .. s0+TS-1
    for (int r = threadIdx.x; r < NRW; r += blockDim.x) {
        const long long s = s0 - QW + r;
        rows[r] = (s >= 0 && s < A.n_steps) ? win_row(A, s) : -1;
    }
    const int sl = threadIdx.x & 31, dg = threadIdx.x >> 5;  // d = dg+1 + 8q
    constexpr int NQ = kGramMaxQW / 8;
    float acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0f;
    __syncthreads();
    for (int k0 = 0; k0 < I; k0 += kGramKC) {
        for (int e = threadIdx.x; e < NRW * kGramKC; e += blockDim.x) {
            const int r = e / kGramKC, kk = e - r * kGramKC;
            const long long row = rows[r];
            xs[r][kk] = (row >= 0 && k0 + kk < I) ? __ldg(A.X + row * I + k0 + kk) : 0.0f;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kGramKC; ++kk) {
            const float xv = xs[QW + sl][kk];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int d = dg + 1 + 8 * q;
                if (d <= QW) acc[q] = fmaf(xv, xs[QW + sl - d][kk], acc[q]);
            }
        }
        __syncthreads();
    }
    const long long s = s0 + sl;
    if (s < A.n_steps) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int d = dg + 1 + 8 * q;
            if (d <= QW) A.coef[s * QW + (d - 1)] = (s - d >= 0) ? A.neg_eta * acc[q] : 0.0f;
        }
    }
}

// ---------------------------------------------------------------------------
// Producer CTA: W0 columns [4p, 4p+4) in registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void win_producer(const WinArgs& A, float* sm, const WinSmem& L) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, D = A.D, P = A.P;
    const int p = blockIdx.x - 1, col = 4 * p;
    const long long n = A.n_steps;
    const int nblk = (int)((n + kWinS - 1) / kWinS);
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    float* red = sm + L.red;
    float4* d0s = reinterpret_cast<float4*>(sm + L.d0s);
    __shared__ long long rk[kWinS], rn[kWinS];  // dataset rows of the update / Y blocks

    float4 w[kWinMaxNR];
#pragma unroll
    for (int m = 0; m < kWinMaxNR; ++m) {
        const int i = tid + kWinThreads * m;
        w[m] = i < I ? *reinterpret_cast<const float4*>(A.W0 + (size_t)i * H + col)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    // Y(b)[u][col..col+3] = x(row_u) . W0[:, col..col+3] with the current registers
    auto compute_y = [&](int b) {
        const int nv = (int)min((long long)kWinS, n - (long long)b * kWinS);
        float acc[4 * kWinS];
#pragma unroll
        for (int e = 0; e < 4 * kWinS; ++e) acc[e] = 0.0f;
#pragma unroll
        for (int u = 0; u < kWinS; ++u) {
            if (u < nv) {
                const float* xr = A.X + rn[u] * I;
#pragma unroll
                for (int m = 0; m < kWinMaxNR; ++m) {
                    const int i = tid + kWinThreads * m;
                    if (i < I) {
                        const float x = __ldg(xr + i);
                        acc[4 * u + 0] = fmaf(x, w[m].x, acc[4 * u + 0]);
                        acc[4 * u + 1] = fmaf(x, w[m].y, acc[4 * u + 1]);
                        acc[4 * u + 2] = fmaf(x, w[m].z, acc[4 * u + 2]);
                        acc[4 * u + 3] = fmaf(x, w[m].w, acc[4 * u + 3]);
                    }
                }
            }
        }
        // 64 values -> 2 per lane (indices 2*lane, 2*lane+1)
        xpose_step<64>(acc, lane, 16);
        xpose_step<32>(acc, lane, 8);
        xpose_step<16>(acc, lane, 4);
        xpose_step<8>(acc, lane, 2);
        xpose_step<4>(acc, lane, 1);
        red[warp * 64 + 2 * lane] = acc[0];
        red[warp * 64 + 2 * lane + 1] = acc[1];
        __syncthreads();
        if (tid < 4 * kWinS) {
            float y = 0.0f;
#pragma unroll
            for (int q = 0; q < kWinWarps; ++q) y += red[q * 64 + tid];
            const int u = tid >> 2, c = tid & 3;
            if (u < nv) __stcg(A.yring + ((size_t)(b % YR) * kWinS + u) * H + col + c, y);
            __threadfence();
        }
        __syncthreads();
        if (tid == 0) red_release_add(A.ycnt + (b % YR), 1u);
    };
    auto stage_rows = [&](long long* dst, int b) {
        if (tid < kWinS) {
            const long long s = (long long)b * kWinS + tid;
            dst[tid] = s < n ? win_row(A, s) : 0;
        }
    };

    const int npro = min(D, nblk);
    for (int b = 0; b < npro; ++b) {
        stage_rows(rn, b);
        __syncthreads();
        compute_y(b);
    }
    for (int k = 0; k < nblk; ++k) {
        if (tid == 0) spin_geq(A.dcnt, (unsigned)(k + 1), A.error);
        __syncthreads();
        const int nv = (int)min((long long)kWinS, n - (long long)k * kWinS);
        if (tid < kWinS) {
            d0s[tid] = tid < nv ? __ldcg(reinterpret_cast<const float4*>(
                                          A.dring + ((size_t)(k % DR) * kWinS + tid) * H + col))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        stage_rows(rk, k);
        const bool do_y = k + D < nblk;
        if (do_y) stage_rows(rn, k + D);
        __syncthreads();
        // the S per-sample updates, reference rounding, in sample order
        for (int u = 0; u < nv; ++u) {
            const float4 d = d0s[u];
            const float* xr = A.X + rk[u] * I;
#pragma unroll
            for (int m = 0; m < kWinMaxNR; ++m) {
                const int i = tid + kWinThreads * m;
                if (i < I) {
                    const float x = __ldg(xr + i);
                    w[m].x = sgd_apply(w[m].x, neg_eta, d.x, x);
                    w[m].y = sgd_apply(w[m].y, neg_eta, d.y, x);
                    w[m].z = sgd_apply(w[m].z, neg_eta, d.z, x);
                    w[m].w = sgd_apply(w[m].w, neg_eta, d.w, x);
                }
            }
        }
        if (do_y) compute_y(k + D);
    }
    (void)P;
#pragma unroll
    for (int m = 0; m < kWinMaxNR; ++m) {
        const int i = tid + kWinThreads * m;
        if (i < I) *reinterpret_cast<float4*>(A.W0 + (size_t)i * H + col) = w[m];
    }
    if (p == 0 && n > 0) {
        const float* xl = A.X + win_row(A, n - 1) * I;
        for (int i = tid; i < I; i += kWinThreads) A.x0[i] = xl[i];
    }
}

// ---------------------------------------------------------------------------
// Chain CTA.
// ---------------------------------------------------------------------------
template <int JPL, int CT>
__device__ __forceinline__ void win_chain(const WinArgs& A, float* sm, const WinSmem& L) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = A.H, D = A.D, HP = L.HP, R = L.R, Rd = L.Rd, QW = A.QW;
    const int HQ = H >> 2, HPQ = HP >> 2;  // float4 per row (used / padded)
    const int C = CT > 0 ? CT : A.C;
    const long long n = A.n_steps;
    const int nblk = (int)((n + kWinS - 1) / kWinS);
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    float* zacc = sm + L.zacc;
    float* ystage = sm + L.ystage;
    float* tstage = sm + L.tstage;
    float* c1stage = sm + L.c1stage;
    float* d0ring = sm + L.d0ring;
    float* pring = sm + L.pring;
    const uint32_t mb = smem_u32(sm + L.mbar);
    auto MB = [&](int idx) { return mb + 8u * (uint32_t)idx; };

    // ---- prologue: zero the rings, init the barriers
    for (int e = tid; e < R * HP; e += kWinThreads) zacc[e] = 0.0f;
    for (int e = tid; e < 2 * kWinS * HP; e += kWinThreads) ystage[e] = 0.0f;
    for (int e = tid; e < 2 * kWinS * kWinCP; e += kWinThreads) tstage[e] = 0.0f;
    for (int e = tid; e < Rd * HP; e += kWinThreads) d0ring[e] = 0.0f;
    if (tid == 0) {
        for (int r = 0; r < kWinRing; ++r) {
            mbar_init(MB(kMbD0 + r), 32);
            mbar_init(MB(kMbRow + r), 32);
        }
        for (int r = 0; r < 2; ++r) {
            mbar_init(MB(kMbYFull + r), 32);
            mbar_init(MB(kMbYFree + r), 32);
        }
        for (int r = 0; r < kWinBlkRing; ++r) mbar_init(MB(kMbBlk + r), 32);
    }
    __syncthreads();
    // rows 0 and 1 need no helper work: complete their row-ready phases so
    // that phase p of ring slot j always means row j + 16p
    if (warp == 0) {
        mbar_arrive_cta(MB(kMbRow + 0));
        mbar_arrive_cta(MB(kMbRow + 1));
    }

    if (warp == kWinCrit) {
        // ================= the serial chain =================
        constexpr int CC = CT > 0 ? CT : kWinCP;
        constexpr int NQ = JPL / 4;
        const int myk = lane >> 1;  // class held after the transpose-reduce
        const bool kval = myk < C;
        float w1[JPL][CC], b0r[JPL], dprev[JPL];
#pragma unroll
        for (int m = 0; m < JPL; ++m) {
            const int j = JPL * lane + m;
#pragma unroll
            for (int k = 0; k < CC; ++k) w1[m][k] = (j < H && k < C) ? A.W1[(size_t)j * C + k] : 0.0f;
            b0r[m] = j < H ? A.b0[j] : 0.0f;
            dprev[m] = 0.0f;
        }
        float b1k = kval ? A.b1[myk] : 0.0f;
        float zl[JPL], al[JPL], zkl = 0.0f, pkl = 0.0f, dkl = 0.0f;
#pragma unroll
        for (int m = 0; m < JPL; ++m) zl[m] = al[m] = 0.0f;
        for (long long s = 0; s < n; ++s) {
            const int b = (int)(s / kWinS), u = (int)(s % kWinS), st = b & 1;
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 0] = clock64();
            if (u == 0) mbar_wait_cta(MB(kMbYFull + st), (uint32_t)((b >> 1) & 1), A.error);
            mbar_wait_cta(MB(kMbRow + (int)(s % kWinRing)), (uint32_t)((s / kWinRing) & 1), A.error);
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 1] = clock64();
            const float c1 = c1stage[st * kWinS + u];
            const float4* zr = reinterpret_cast<const float4*>(zacc + (size_t)(s % R) * HP) + lane * NQ;
            const float4* yr = reinterpret_cast<const float4*>(ystage + (size_t)(st * kWinS + u) * HP) + lane * NQ;
            float z[JPL], a[JPL];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 za = zr[q], ya = yr[q];
                z[4 * q + 0] = fmaf(c1, dprev[4 * q + 0], za.x + ya.x) + b0r[4 * q + 0];
                z[4 * q + 1] = fmaf(c1, dprev[4 * q + 1], za.y + ya.y) + b0r[4 * q + 1];
                z[4 * q + 2] = fmaf(c1, dprev[4 * q + 2], za.z + ya.z) + b0r[4 * q + 2];
                z[4 * q + 3] = fmaf(c1, dprev[4 * q + 3], za.w + ya.w) + b0r[4 * q + 3];
            }
#pragma unroll
            for (int m = 0; m < JPL; ++m) a[m] = tanhf(z[m]);
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 2] = clock64();
            // partial logits of this lane's hidden units, then the transpose-reduce
            float P[kWinCP];
#pragma unroll
            for (int k = 0; k < kWinCP; ++k) {
                float acc = 0.0f;
                if (k < CC) {
#pragma unroll
                    for (int m = 0; m < JPL; ++m) acc = fmaf(a[m], w1[m][k], acc);
                }
                P[k] = acc;
            }
            xpose_step<16>(P, lane, 16);
            xpose_step<8>(P, lane, 8);
            xpose_step<4>(P, lane, 4);
            xpose_step<2>(P, lane, 2);
            float zk = P[0] + __shfl_xor_sync(0xffffffffu, P[0], 1);
            zk = sadd(zk, b1k);
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 3] = clock64();
            float mx = kval ? zk : -INFINITY;
#pragma unroll
            for (int o = 2; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float e = kval ? expf(zk - mx) : 0.0f;
            float sum = e;
#pragma unroll
            for (int o = 2; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const float pk = __fdiv_rn(e, sum);
            const float tk = kval ? tstage[(st * kWinS + u) * kWinCP + myk] : 0.0f;
            const float dk = kval ? ssub(pk, tk) : 0.0f;
            float d1[CC];
#pragma unroll
            for (int k = 0; k < CC; ++k) d1[k] = __shfl_sync(0xffffffffu, dk, 2 * k);
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 4] = clock64();
            // hidden deltas with the pre-update W1
            float d0v[JPL];
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                float acc = 0.0f;
#pragma unroll
                for (int k = 0; k < CC; ++k) acc = fmaf(d1[k], w1[m][k], acc);
                d0v[m] = tanh_grad(a[m], acc);
            }
            float4* dr = reinterpret_cast<float4*>(d0ring + (size_t)(s % Rd) * HP) + lane * NQ;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                dr[q] = make_float4(d0v[4 * q], d0v[4 * q + 1], d0v[4 * q + 2], d0v[4 * q + 3]);
            if (kval && !(lane & 1)) pring[(size_t)(s % Rd) * kWinCP + myk] = pk;
            mbar_arrive_cta(MB(kMbD0 + (int)(s % kWinRing)));
            if (u == kWinS - 1 || s == n - 1) {
                mbar_arrive_cta(MB(kMbBlk + b % kWinBlkRing));
                mbar_arrive_cta(MB(kMbYFree + st));
            }
            if (A.trace && lane == 0 && s < kTraceSamples) A.trace[s * kTracePhases + 5] = clock64();
            // updates of sample s (reference rounding)
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
#pragma unroll
                for (int k = 0; k < CC; ++k) w1[m][k] = sgd_apply(w1[m][k], neg_eta, d1[k], a[m]);
                b0r[m] = sadd(b0r[m], smul(neg_eta, d0v[m]));
                dprev[m] = d0v[m];
            }
            b1k = sadd(b1k, smul(neg_eta, dk));
            if (s == n - 1) {
#pragma unroll
                for (int m = 0; m < JPL; ++m) {
                    zl[m] = z[m];
                    al[m] = a[m];
                }
                zkl = zk;
                pkl = pk;
                dkl = dk;
            }
        }
        if (n > 0) {
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                const int j = JPL * lane + m;
                if (j < H) {
#pragma unroll
                    for (int k = 0; k < CC; ++k)
                        if (k < C) A.W1[(size_t)j * C + k] = w1[m][k];
                    A.b0[j] = b0r[m];
                    A.z0[j] = zl[m];
                    A.a0[j] = al[m];
                    A.d0[j] = dprev[m];
                    A.db0[j] = smul(neg_eta, dprev[m]);
                    A.x1[j] = al[m];
                }
            }
            if (kval && !(lane & 1)) {
                A.b1[myk] = b1k;
                A.z1[myk] = zkl;
                A.a1[myk] = pkl;
                A.d1[myk] = dkl;
                A.db1[myk] = smul(neg_eta, dkl);
            }
        }
    } else if (warp == kWinLoad) {
        // ================= loader: Y(b), targets, c(s,1) =================
        for (int b = 0; b < nblk; ++b) {
            const int st = b & 1;
            if (b >= 2) mbar_wait_cta(MB(kMbYFree + st), (uint32_t)(((b - 2) >> 1) & 1), A.error);
            spin_geq(A.ycnt + (b % YR), (unsigned)(A.P * (b / YR + 1)), A.error);
            const int nv = (int)min((long long)kWinS, n - (long long)b * kWinS);
            const float4* src = reinterpret_cast<const float4*>(A.yring + (size_t)(b % YR) * kWinS * H);
            float4* dst = reinterpret_cast<float4*>(ystage + (size_t)st * kWinS * HP);
            for (int e = lane; e < nv * HQ; e += 32) {
                const int u = e / HQ, q = e - u * HQ;
                dst[u * HPQ + q] = __ldcg(src + u * HQ + q);
            }
            for (int e = lane; e < nv * C; e += 32) {
                const int u = e / C, k = e - u * C;
                const long long row = win_row(A, (long long)b * kWinS + u);
                tstage[(st * kWinS + u) * kWinCP + k] = __ldg(A.T + row * C + k);
            }
            if (lane < kWinS)
                c1stage[st * kWinS + lane] = lane < nv ? __ldg(A.coef + ((long long)b * kWinS + lane) * QW) : 0.0f;
            mbar_arrive_cta(MB(kMbYFull + st));
        }
    } else if (warp == kWinPub) {
        // ================= publisher: d0 blocks to L2, loss/accuracy =================
        double loss_acc = (lane == 0 && A.loss_sum) ? *A.loss_sum : 0.0;
        unsigned long long correct_acc = 0;
        for (int k = 0; k < nblk; ++k) {
            mbar_wait_cta(MB(kMbBlk + k % kWinBlkRing), (uint32_t)((k / kWinBlkRing) & 1), A.error);
            const int nv = (int)min((long long)kWinS, n - (long long)k * kWinS);
            float4* dst = reinterpret_cast<float4*>(A.dring + (size_t)(k % DR) * kWinS * H);
            for (int e = lane; e < nv * HQ; e += 32) {
                const int u = e / HQ, q = e - u * HQ;
                const long long s = (long long)k * kWinS + u;
                __stcg(dst + u * HQ + q, reinterpret_cast<const float4*>(d0ring + (size_t)(s % Rd) * HP)[q]);
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) red_release_add(A.dcnt, 1u);
            if (lane == 0 && (A.loss_sum || A.correct)) {
                for (int u = 0; u < nv; ++u) {
                    const long long s = (long long)k * kWinS + u;
                    const float* tc = A.T + win_row(A, s) * C;
                    const float* pl = pring + (size_t)(s % Rd) * kWinCP;
                    float loss = 0.0f;
                    int bp = 0, btg = 0;
                    for (int o = 0; o < C; ++o) {
                        const float to = __ldg(tc + o);
                        if (to != 0.0f) {
                            const float q = pl[o] < 1e-12f ? 1e-12f : pl[o];
                            loss = ssub(loss, smul(to, logf(q)));
                        }
                        if (pl[o] > pl[bp]) bp = o;
                        if (to > __ldg(tc + btg)) btg = o;
                    }
                    loss_acc = __dadd_rn(loss_acc, (double)loss);
                    correct_acc += bp == btg;
                }
            }
        }
        if (lane == 0) {
            if (A.loss_sum) *A.loss_sum = loss_acc;
            if (A.correct) *A.correct += correct_acc;
        }
    } else {
        // ================= helpers: window corrections =================
        const int w = warp;
        float cf[kWinMaxMine];
        for (long long s = 0; s < n; ++s) {
            const long long b = s / kWinS;
            const long long last = min(n - 1, (b + D) * kWinS - 1);
            // first owned row >= s+2
            const long long f0 = s + 2;
            const long long first = f0 + ((w - (int)(f0 % kWinHelpers)) + kWinHelpers) % kWinHelpers;
#pragma unroll
            for (int i = 0; i < kWinMaxMine; ++i) {
                const long long r = first + (long long)i * kWinHelpers;
                cf[i] = r <= last ? __ldg(A.coef + r * QW + (r - s - 1)) : 0.0f;
            }
            mbar_wait_cta(MB(kMbD0 + (int)(s % kWinRing)), (uint32_t)((s / kWinRing) & 1), A.error);
            const float4* dv = reinterpret_cast<const float4*>(d0ring + (size_t)(s % Rd) * HP);
            // urgent row s+2 first (if owned), then signal it
            if (first == f0 && f0 <= last) {
                float4* zr = reinterpret_cast<float4*>(zacc + (size_t)(f0 % R) * HP);
                for (int q = lane; q < HQ; q += 32) {
                    const float4 d = dv[q];
                    float4 z = zr[q];
                    z.x = fmaf(cf[0], d.x, z.x);
                    z.y = fmaf(cf[0], d.y, z.y);
                    z.z = fmaf(cf[0], d.z, z.z);
                    z.w = fmaf(cf[0], d.w, z.w);
                    zr[q] = z;
                }
            }
            if (first == f0 && f0 < n) mbar_arrive_cta(MB(kMbRow + (int)(f0 % kWinRing)));
            const int i0 = first == f0 ? 1 : 0;
            for (int q = lane; q < HQ; q += 32) {
                const float4 d = dv[q];
#pragma unroll
                for (int i = 0; i < kWinMaxMine; ++i) {
                    const long long r = first + (long long)i * kWinHelpers;
                    if (i >= i0 && r <= last) {
                        float4* zr = reinterpret_cast<float4*>(zacc + (size_t)(r % R) * HP) + q;
                        float4 z = *zr;
                        z.x = fmaf(cf[i], d.x, z.x);
                        z.y = fmaf(cf[i], d.y, z.y);
                        z.z = fmaf(cf[i], d.z, z.z);
                        z.w = fmaf(cf[i], d.w, z.w);
                        *zr = z;
                    }
                }
            }
            // row s has been consumed: its slot now belongs to row s + R
            if ((int)(s % kWinHelpers) == w) {
                float4* zr = reinterpret_cast<float4*>(zacc + (size_t)(s % R) * HP);
                for (int q = lane; q < HQ; q += 32) zr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
}

template <int JPL, int CT>
__global__ void __launch_bounds__(kWinThreads, 1) k_sgd_window(WinArgs A) {
    extern __shared__ __align__(16) float sm[];
    const WinSmem L(32 * JPL, A.D);
    if (blockIdx.x == 0)
        win_chain<JPL, CT>(A, sm, L);
    else
        win_producer(A, sm, L);
}

}  // namespace lane_b200
