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
// (stored forward: c(r, r-s) = coef[s][r-s-1], contiguous for one source s)
//
// Numerics: FAST (the forward dot products are reassociated); the weights
// receive exactly the reference's per-sample update sequence given d0.
#pragma once

#include "common.cuh"
#include "sgd_persistent.cuh"

namespace lane_b200 {

constexpr int kWinS = 16;                    // samples per block
constexpr int kWinHelpers = 4;               // helper warps
constexpr int kWinWarps = 10;                // max warps per CTA (four chain warps)
constexpr int kWinThreads = 32 * kWinWarps;  // 256
// CTA size: 7 warps with one chain warp, 8 with two
template <int NCW>
constexpr int win_threads() { return NCW == 4 ? 320 : NCW == 2 ? 256 : 224; }
// Warp roles.  Warps share a sub-partition (SMSP) when their ids are equal mod
// 4: SMSP0 = helper 0 + helper 2 (warp 4), SMSP1 = helper 1 + helper 3 (warp
// 5), SMSP2 = chain warp 2 + publisher (6), SMSP3 = chain warp 3 + loader (7).
// The publisher and loader mostly sleep on mbarriers / spin on L2 counters.
// NCW = 1 (7 warps): helpers 0,1,2,4; chain 3 (alone on SMSP3); publisher 5;
//   loader 6.
// NCW = 2 (8 warps): helpers 0,1,4,5; chain 2,3; publisher 6; loader 7.
// NCW = 4 (10 warps): chain 0..3 (one per SMSP); helpers 4..7; publisher 8;
//   loader 9.
template <int NCW>
__device__ __forceinline__ int win_loader_warp() { return NCW == 4 ? 9 : NCW == 2 ? 7 : 6; }
template <int NCW>
__device__ __forceinline__ int win_pub_warp() { return NCW == 4 ? 8 : NCW == 2 ? 6 : 5; }
// helper index 0..3, or -1
template <int NCW>
__device__ __forceinline__ int win_helper_index(int warp) {
    if (NCW == 4) return (warp >= 4 && warp < 8) ? warp - 4 : -1;
    if (NCW == 2) return (warp == 0 || warp == 1) ? warp : (warp == 4 || warp == 5) ? warp - 2 : -1;
    return warp < 3 ? warp : warp == 4 ? 3 : -1;
}
// chain warp index (0..NCW-1) or -1: NCW = 1 uses warp 3 (warp 2 idles)
template <int NCW>
__device__ __forceinline__ int win_chain_index(int warp) {
    if (NCW == 4) return warp < 4 ? warp : -1;
    return NCW == 2 ? ((warp == 2 || warp == 3) ? warp - 2 : -1) : (warp == 3 ? 0 : -1);
}
// vector load/store of JPL consecutive floats (JPL = 2 or 4)
template <int JPL>
__device__ __forceinline__ void vld(const float* p, float* v) {
    if constexpr (JPL % 4 == 0) {
#pragma unroll
        for (int i = 0; i < JPL / 4; ++i) {
            const float4 q = reinterpret_cast<const float4*>(p)[i];
            v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
        }
    } else {
        static_assert(JPL == 2, "JPL must be 2 or a multiple of 4");
        const float2 q = *reinterpret_cast<const float2*>(p);
        v[0] = q.x; v[1] = q.y;
    }
}
template <int JPL>
__device__ __forceinline__ void vst(float* p, const float* v) {
    if constexpr (JPL % 4 == 0) {
#pragma unroll
        for (int i = 0; i < JPL / 4; ++i)
            reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    }
}
constexpr int kWinMaxD = 6;
constexpr int kWinRing = 16;                 // d0-ready / row-ready mbarrier rings
constexpr int kWinBlkRing = 8;               // block-done mbarrier ring (> D)
constexpr int kWinMaxNR = 4;                 // producer: W0 rows per thread (I <= 4 * 352)
constexpr int kWinCP = 16;                   // classes padded for the transpose-reduce
constexpr int kWinMaxCS = 16;                // chain CTAs per cluster

struct WinArgs {
    int I, H, C, D, P, QW;
    int KS, RPC;  // producers: row splits per column group, rows per split
    int QPC;      // producers: column quads per CTA (P = ceil(H/4 / QPC) * KS active producers)
    int CS;       // chain CTAs (one thread-block cluster); producers are CTAs CS..
    const float* X;
    const float* T;
    const uint32_t* order;  // stream order (offset to this launch) or null
    int n;                  // dataset rows (< 2^31)
    int n_steps;            // samples in this launch (<= 2^18)
    int base;               // first stream position mod n (no order: row = (base + s) % n)
    float neg_eta;
    float *W0, *b0, *W1, *b1;
    float* coef;        // [n_steps][QW]: -eta x(s).x(s+d) at [s][d-1] (forward band)
    float* yring;       // [D+1][KS][S][H] partial Y per row split
    float* dring;       // [D+1][S][H]
    unsigned* ycnt;     // [D+1] monotonic producer arrivals per Y slot
    unsigned* dcnt;     // published d0 blocks
    float *x0, *z0, *a0, *d0, *db0;
    float *x1, *z1, *a1, *d1, *db1;
    double* loss_sum;
    unsigned long long* correct;
    int* error;
    unsigned long long* trace;
    int trace_base;  // first traced stream position
};

struct WinSmem {
    int HP, R, Rd, Rdh;  // Rdh: rows of the shared-memory d0 ring (helpers, publisher)
    size_t zacc, ystage, tstage, coefs, d0ring, pring, red, d0s, rowflag, gat, mbar, total;
    // HP_: padded hidden slice per chain CTA; Hs: the slice width (H / CS)
    // direct: the chain also writes d0 rows straight to the L2 ring (cluster
    // chains), so the shared ring only covers the helpers' lag (16 rows)
    __host__ __device__ WinSmem(int HP_, int D, int KS, int Hs, int NCW, bool direct = false) : HP(HP_) {
        R = D * kWinS;
        Rd = (D + 1) * kWinS;
        Rdh = direct ? kWinS : Rd;
        size_t o = 0;
        auto take = [&](size_t nf) {
            size_t at = o;
            o += (nf + 3) & ~size_t(3);
            return at;
        };
        zacc = take((size_t)R * HP);
        ystage = take(2 * (size_t)KS * kWinS * Hs);  // [buffer][ks][u][Hs] (TMA bulk copies)
        tstage = take(2 * kWinS * kWinCP);
        coefs = take((size_t)Rd * D * kWinS);  // forward band rows of source s, slot s % Rd
        d0ring = take((size_t)Rdh * HP);
        pring = take((size_t)Rd * kWinCP);
        red = take(kWinCP * (32 * NCW + 4) + 4 * NCW * kWinCP);  // partials, halves x2, logits, exps
        d0s = take(kWinS * 4);
        rowflag = take(R);
        gat = take(2 * kWinMaxCS * kWinCP);  // [parity][rank][class]: cluster logit exchange
        mbar = take(2 * (kWinRing + 6 + kWinBlkRing));
        total = o * sizeof(float);
    }
};

// mbarrier indices (u64 slots)
constexpr int kMbD0 = 0, kMbYFull = kWinRing, kMbYFree = kWinRing + 2, kMbBlk = kWinRing + 4,
              kMbXch = kWinRing + 4 + kWinBlkRing;  // 2 exchange barriers (by sample parity)

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
__device__ __forceinline__ void mbar_wait_slow(uint32_t a, uint32_t parity, int* err) {
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

// dataset row of stream position s (32-bit unsigned arithmetic: no 64-bit
// division subroutine anywhere in these kernels)
__device__ __forceinline__ long long win_row(const WinArgs& A, int s) {
    return A.order ? (long long)A.order[s] : (long long)(((unsigned)A.base + (unsigned)s) % (unsigned)A.n);
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
// Banded Gram pre-pass (forward band): coef[s][d-1] = -eta * (x(s) . x(s+d)),
// d = 1..QW (0 past the end of the stream), so that the coefficients a new
// d0(s) needs for every later row r = s+d are contiguous.  One CTA per 32
// stream positions; K streamed through shared memory in 32-float chunks.
// ---------------------------------------------------------------------------
constexpr int kGramTS = 32, kGramKC = 64, kGramMaxQW = 96;

// NQ = ceil(QW / 8): thread (sl, dg) accumulates d = dg+1, dg+9, ... <= QW.
// K chunks of 64 floats, loaded as float4 (I % 4 == 0) one chunk ahead in
// registers, so the global latency hides under the previous chunk's FMAs.
template <int NQ>
__global__ void __launch_bounds__(256) k_gram_band(WinArgs A) {
    constexpr int kRows = kGramTS + 8 * NQ;            // rows s0 .. s0+TS+QW-1 (QW <= 8 NQ)
    constexpr int kLd = (kRows * kGramKC / 4 + 255) / 256;  // float4 loads per thread per chunk
    __shared__ float xs[kRows][kGramKC + 1];
    __shared__ long long rows[kRows];
    const int QW = A.QW, I = A.I;
    const int s0 = blockIdx.x * kGramTS;
    const int NRW = kGramTS + QW;
    for (int r = threadIdx.x; r < kRows; r += blockDim.x) {
        const int s = s0 + r;
        rows[r] = (r < NRW && s < A.n_steps) ? win_row(A, s) : -1;
    }
    const int sl = threadIdx.x & 31, dg = threadIdx.x >> 5;
    float acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0f;
    __syncthreads();
    const bool vec = (I & 3) == 0;
    float4 pf[kLd];
    auto load = [&](int k0) {
#pragma unroll
        for (int l = 0; l < kLd; ++l) {
            const int e = threadIdx.x + 256 * l;  // (row, quad) = (e / 16, e % 16)
            const int r = e >> 4, kk = (e & 15) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            const long long row = r < kRows ? rows[r] : -1;
            if (row >= 0) {
                const float* src = A.X + row * I + k0 + kk;
                if (vec && k0 + kk + 3 < I) {
                    v = __ldg(reinterpret_cast<const float4*>(src));
                } else {
                    if (k0 + kk + 0 < I) v.x = __ldg(src + 0);
                    if (k0 + kk + 1 < I) v.y = __ldg(src + 1);
                    if (k0 + kk + 2 < I) v.z = __ldg(src + 2);
                    if (k0 + kk + 3 < I) v.w = __ldg(src + 3);
                }
            }
            pf[l] = v;
        }
    };
    load(0);
    for (int k0 = 0; k0 < I; k0 += kGramKC) {
#pragma unroll
        for (int l = 0; l < kLd; ++l) {
            const int e = threadIdx.x + 256 * l;
            const int r = e >> 4, kk = (e & 15) * 4;
            if (r < kRows) {
                xs[r][kk + 0] = pf[l].x;
                xs[r][kk + 1] = pf[l].y;
                xs[r][kk + 2] = pf[l].z;
                xs[r][kk + 3] = pf[l].w;
            }
        }
        __syncthreads();
        if (k0 + kGramKC < I) load(k0 + kGramKC);
#pragma unroll 8
        for (int kk = 0; kk < kGramKC; ++kk) {
            const float xv = xs[sl][kk];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = fmaf(xv, xs[sl + dg + 1 + 8 * q][kk], acc[q]);
        }
        __syncthreads();
    }
    const int s = s0 + sl;
    if (s < A.n_steps) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int d = dg + 1 + 8 * q;
            if (d <= QW) A.coef[(size_t)s * QW + (d - 1)] = (s + d < A.n_steps) ? A.neg_eta * acc[q] : 0.0f;
        }
    }
}

// ---------------------------------------------------------------------------
// Producer CTAs.  Producer (pc, ks) owns W0 columns [4 pc QPC, 4 (pc+1) QPC)
// (QPC column quads) x rows [ks*RPC, ks*RPC + RPC) in registers for the whole
// stream.  The X rows of the last D+2 blocks of its row range sit in a
// shared-memory ring, filled by cp.async one iteration ahead: block k's rows
// arrive for Y(k) (iteration k-D) and are reused for block k's weight update
// (iteration k).  Per block k: acquire d0 of block k (all CS chain CTAs), apply
// its S per-sample updates with the reference's exact rounding
// (w + (-eta * (d0 * x)), sample by sample), then publish the partial Y(k+D)
// of this row range; the chain sums the KS partials of a column in a fixed
// order.
// ---------------------------------------------------------------------------
constexpr int kWinMaxQPC = 4;  // column quads per producer CTA

struct ProdSmem {
    int RPCp, NB;
    size_t xr, d0s, red, total;
    __host__ __device__ ProdSmem(int RPC, int D) {
        RPCp = (RPC + 3) & ~3;
        NB = D + 2;
        size_t o = 0;
        auto take = [&](size_t nf) {
            size_t at = o;
            o += (nf + 3) & ~size_t(3);
            return at;
        };
        xr = take((size_t)NB * kWinS * RPCp);
        d0s = take(kWinS * 8 * 4);  // [u][quad] float4, up to 8 quads
        red = take(kWinWarps * 64);
        total = o * sizeof(float);
    }
};

template <int NT, int MQ, int NR>
__device__ __forceinline__ void win_producer(const WinArgs& A, float* sm) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, D = A.D, KS = A.KS, RPC = A.RPC, QPC = A.QPC;
    const int pid = blockIdx.x - A.CS;
    const int pc = pid / KS, ks = pid - pc * KS;
    const int q0 = pc * QPC, nq = max(0, min(QPC, (H >> 2) - q0));  // this CTA's column quads
    if (nq == 0) return;                                           // padding CTA of the cluster grid
    const int i0 = ks * RPC, nr = max(0, min(I, i0 + RPC) - i0);
    const int n = A.n_steps;
    const int nblk = (n + kWinS - 1) / kWinS;
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    const ProdSmem L(RPC, D);
    const int RPCp = L.RPCp, NB = L.NB;
    float* xr = sm + L.xr;
    float* red = sm + L.red;
    float4* d0s = reinterpret_cast<float4*>(sm + L.d0s);  // [u][quad]
    const bool vec = ((I & 3) == 0) && ((i0 & 3) == 0) && ((nr & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(A.X) & 15) == 0);

    float4 w[MQ][NR];
#pragma unroll
    for (int qi = 0; qi < MQ; ++qi)
#pragma unroll
        for (int m = 0; m < NR; ++m) {
            const int li = tid + NT * m;
            w[qi][m] = (qi < nq && li < nr)
                           ? *reinterpret_cast<const float4*>(A.W0 + (size_t)(i0 + li) * H + 4 * (q0 + qi))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    // X rows [i0, i0+nr) of block blk -> ring slot blk % NB (cp.async, no wait)
    auto prefetch = [&](int blk) {
        float* dst = xr + (size_t)(blk % NB) * kWinS * RPCp;
        const int s0 = blk * kWinS, nv = min(kWinS, n - s0);
        if (vec) {
            const int nq4 = nr >> 2;
            for (int e = tid; e < nv * nq4; e += NT) {
                const int u = e / nq4, q = e - u * nq4;
                cp_async16(dst + u * RPCp + 4 * q, A.X + win_row(A, s0 + u) * I + i0 + 4 * q);
            }
        } else {
            for (int e = tid; e < nv * nr; e += NT) {
                const int u = e / nr, q = e - u * nr;
                cp_async4(dst + u * RPCp + q, A.X + win_row(A, s0 + u) * I + i0 + q);
            }
        }
    };
    // partial Y(blk)[u][cols] over this row range from the current registers,
    // one column quad at a time (64 accumulators per thread)
    auto compute_y = [&](int blk) {
        const float* xb = xr + (size_t)(blk % NB) * kWinS * RPCp;
        const int nv = min(kWinS, n - blk * kWinS);
#pragma unroll
        for (int qi = 0; qi < MQ; ++qi) {
            if (qi >= nq) break;
            float acc[4 * kWinS];
#pragma unroll
            for (int e = 0; e < 4 * kWinS; ++e) acc[e] = 0.0f;
#pragma unroll
            for (int m = 0; m < NR; ++m) {
                const int li = tid + NT * m;
                if (li < nr) {
#pragma unroll
                    for (int u = 0; u < kWinS; ++u) {
                        const float x = u < nv ? xb[u * RPCp + li] : 0.0f;
                        acc[4 * u + 0] = fmaf(x, w[qi][m].x, acc[4 * u + 0]);
                        acc[4 * u + 1] = fmaf(x, w[qi][m].y, acc[4 * u + 1]);
                        acc[4 * u + 2] = fmaf(x, w[qi][m].z, acc[4 * u + 2]);
                        acc[4 * u + 3] = fmaf(x, w[qi][m].w, acc[4 * u + 3]);
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
                for (int q = 0; q < NT / 32; ++q) y += red[q * 64 + tid];
                const int u = tid >> 2, c = tid & 3;
                if (u < nv)
                    __stcg(A.yring + (((size_t)(blk % YR) * KS + ks) * kWinS + u) * H + 4 * (q0 + qi) + c, y);
            }
            __syncthreads();  // red reuse
        }
        // each of the two writer warps releases its own stores
        if (tid < 4 * kWinS) {
            __syncwarp();
            if (lane == 0) red_release_add(A.ycnt + (blk % YR), 1u);
        }
    };

    const int npro = min(D, nblk);
    for (int blk = 0; blk <= npro && blk < nblk; ++blk) prefetch(blk);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int blk = 0; blk < npro; ++blk) compute_y(blk);
    for (int k = 0; k < nblk; ++k) {
        const int nv = min(kWinS, n - k * kWinS);
        if (k + D + 1 < nblk) prefetch(k + D + 1);  // slot of block k-1: retired
        cp_async_commit();
        if (tid == 0) spin_geq(A.dcnt, (unsigned)(A.CS * (k + 1)), A.error);
        __syncthreads();
        if (tid < kWinS * MQ) {
            const int u = tid / MQ, qi = tid - u * MQ;
            d0s[tid] = (u < nv && qi < nq) ? __ldcg(reinterpret_cast<const float4*>(
                                                 A.dring + ((size_t)(k % DR) * kWinS + u) * H + 4 * (q0 + qi)))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        cp_async_wait<1>();  // block k+D's rows (prefetched last iteration) have landed
        __syncthreads();
        // the S per-sample updates, reference rounding, in sample order
        const float* xb = xr + (size_t)(k % NB) * kWinS * RPCp;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
            const int li = tid + NT * m;
            if (li < nr) {
#pragma unroll
                for (int u = 0; u < kWinS; ++u) {
                    if (u < nv) {
                        const float x = xb[u * RPCp + li];
#pragma unroll
                        for (int qi = 0; qi < MQ; ++qi) {
                            if (qi < nq) {
                                const float4 d = d0s[u * MQ + qi];
                                w[qi][m].x = sgd_apply(w[qi][m].x, neg_eta, d.x, x);
                                w[qi][m].y = sgd_apply(w[qi][m].y, neg_eta, d.y, x);
                                w[qi][m].z = sgd_apply(w[qi][m].z, neg_eta, d.z, x);
                                w[qi][m].w = sgd_apply(w[qi][m].w, neg_eta, d.w, x);
                            }
                        }
                    }
                }
            }
        }
        if (k + D < nblk) compute_y(k + D);
        __syncthreads();  // ring slot / d0s / red reuse
    }
    cp_async_wait<0>();
#pragma unroll
    for (int qi = 0; qi < MQ; ++qi)
#pragma unroll
        for (int m = 0; m < NR; ++m) {
            const int li = tid + NT * m;
            if (qi < nq && li < nr)
                *reinterpret_cast<float4*>(A.W0 + (size_t)(i0 + li) * H + 4 * (q0 + qi)) = w[qi][m];
        }
    if (pid == 0 && n > 0) {
        const float* xl = A.X + win_row(A, n - 1) * I;
        for (int i = tid; i < I; i += NT) A.x0[i] = xl[i];
    }
}

// Producer with its W0 slice in SHARED memory (very wide layers, > 8 column
// quads per CTA): quad-major [quad][row] float4.  Per block, one pass per
// quad: load the thread's row-quads, apply the S updates (reference rounding),
// store them back and, with the updated values still in registers, add this
// quad's contribution to Y(k+D).
constexpr int kWinSmemQPC = 32;
struct ProdSmemS {
    int RPCp, NB;
    size_t xr, d0s, red, wsm, total;
    __host__ __device__ ProdSmemS(int RPC, int D, int QPC) {
        RPCp = (RPC + 3) & ~3;
        NB = D + 2;
        size_t o = 0;
        auto take = [&](size_t nf) {
            size_t at = o;
            o += (nf + 3) & ~size_t(3);
            return at;
        };
        xr = take((size_t)NB * kWinS * RPCp);
        d0s = take(kWinS * kWinSmemQPC * 4);
        red = take(kWinWarps * 64);
        wsm = take((size_t)QPC * RPCp * 4);
        total = o * sizeof(float);
    }
};

template <int NT, int NR>
__device__ __forceinline__ void win_producer_smem(const WinArgs& A, float* sm) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, D = A.D, KS = A.KS, RPC = A.RPC, QPC = A.QPC;
    const int pid = blockIdx.x - A.CS;
    const int pc = pid / KS, ks = pid - pc * KS;
    const int q0 = pc * QPC, nq = max(0, min(QPC, (H >> 2) - q0));
    if (nq == 0) return;
    const int i0 = ks * RPC, nr = max(0, min(I, i0 + RPC) - i0);
    const int n = A.n_steps;
    const int nblk = (n + kWinS - 1) / kWinS;
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    const ProdSmemS L(RPC, D, QPC);
    const int RPCp = L.RPCp, NB = L.NB;
    float* xr = sm + L.xr;
    float* red = sm + L.red;
    float4* d0s = reinterpret_cast<float4*>(sm + L.d0s);  // [u][quad]
    float4* wsm = reinterpret_cast<float4*>(sm + L.wsm);  // [quad][row]
    const bool vec = ((I & 3) == 0) && ((i0 & 3) == 0) && ((nr & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(A.X) & 15) == 0);
    for (int e = tid; e < nq * RPCp; e += NT) {
        const int qi = e / RPCp, li = e - qi * RPCp;
        wsm[e] = li < nr ? *reinterpret_cast<const float4*>(A.W0 + (size_t)(i0 + li) * H + 4 * (q0 + qi))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto prefetch = [&](int blk) {
        float* dst = xr + (size_t)(blk % NB) * kWinS * RPCp;
        const int s0 = blk * kWinS, nv = min(kWinS, n - s0);
        if (vec) {
            const int nq4 = nr >> 2;
            for (int e = tid; e < nv * nq4; e += NT) {
                const int u = e / nq4, q = e - u * nq4;
                cp_async16(dst + u * RPCp + 4 * q, A.X + win_row(A, s0 + u) * I + i0 + 4 * q);
            }
        } else {
            for (int e = tid; e < nv * nr; e += NT) {
                const int u = e / nr, q = e - u * nr;
                cp_async4(dst + u * RPCp + q, A.X + win_row(A, s0 + u) * I + i0 + q);
            }
        }
    };
    // one quad: optional update with block ku's d0 (nvu samples), optional
    // Y(ky) contribution from the resulting weights
    auto quad_pass = [&](int qi, int ku, int nvu, int ky) {
        float4 w[NR];
#pragma unroll
        for (int m = 0; m < NR; ++m) {
            const int li = tid + NT * m;
            w[m] = li < nr ? wsm[qi * RPCp + li] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (ku >= 0) {
            const float* xb = xr + (size_t)(ku % NB) * kWinS * RPCp;
#pragma unroll
            for (int m = 0; m < NR; ++m) {
                const int li = tid + NT * m;
                if (li < nr) {
#pragma unroll
                    for (int u = 0; u < kWinS; ++u) {
                        if (u < nvu) {
                            const float x = xb[u * RPCp + li];
                            const float4 d = d0s[u * kWinSmemQPC + qi];
                            w[m].x = sgd_apply(w[m].x, neg_eta, d.x, x);
                            w[m].y = sgd_apply(w[m].y, neg_eta, d.y, x);
                            w[m].z = sgd_apply(w[m].z, neg_eta, d.z, x);
                            w[m].w = sgd_apply(w[m].w, neg_eta, d.w, x);
                        }
                    }
                    wsm[qi * RPCp + li] = w[m];
                }
            }
        }
        if (ky < 0) return;
        const float* xb = xr + (size_t)(ky % NB) * kWinS * RPCp;
        const int nv = min(kWinS, n - ky * kWinS);
        float acc[4 * kWinS];
#pragma unroll
        for (int e = 0; e < 4 * kWinS; ++e) acc[e] = 0.0f;
#pragma unroll
        for (int m = 0; m < NR; ++m) {
            const int li = tid + NT * m;
            if (li < nr) {
#pragma unroll
                for (int u = 0; u < kWinS; ++u) {
                    const float x = u < nv ? xb[u * RPCp + li] : 0.0f;
                    acc[4 * u + 0] = fmaf(x, w[m].x, acc[4 * u + 0]);
                    acc[4 * u + 1] = fmaf(x, w[m].y, acc[4 * u + 1]);
                    acc[4 * u + 2] = fmaf(x, w[m].z, acc[4 * u + 2]);
                    acc[4 * u + 3] = fmaf(x, w[m].w, acc[4 * u + 3]);
                }
            }
        }
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
            for (int q = 0; q < NT / 32; ++q) y += red[q * 64 + tid];
            const int u = tid >> 2, c = tid & 3;
            if (u < nv) __stcg(A.yring + (((size_t)(ky % YR) * KS + ks) * kWinS + u) * H + 4 * (q0 + qi) + c, y);
        }
        __syncthreads();  // red reuse
    };
    auto release_y = [&](int blk) {
        if (tid < 4 * kWinS) {
            __syncwarp();
            if (lane == 0) red_release_add(A.ycnt + (blk % YR), 1u);
        }
    };

    const int npro = min(D, nblk);
    for (int blk = 0; blk <= npro && blk < nblk; ++blk) prefetch(blk);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int blk = 0; blk < npro; ++blk) {
        for (int qi = 0; qi < nq; ++qi) quad_pass(qi, -1, 0, blk);
        release_y(blk);
    }
    for (int k = 0; k < nblk; ++k) {
        const int nv = min(kWinS, n - k * kWinS);
        if (k + D + 1 < nblk) prefetch(k + D + 1);  // slot of block k-1: retired
        cp_async_commit();
        if (tid == 0) spin_geq(A.dcnt, (unsigned)(A.CS * (k + 1)), A.error);
        __syncthreads();
        for (int e = tid; e < kWinS * kWinSmemQPC; e += NT) {
            const int u = e / kWinSmemQPC, qi = e - u * kWinSmemQPC;
            d0s[e] = (u < nv && qi < nq) ? __ldcg(reinterpret_cast<const float4*>(
                                               A.dring + ((size_t)(k % DR) * kWinS + u) * H + 4 * (q0 + qi)))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        cp_async_wait<1>();  // block k+D's rows (prefetched last iteration) have landed
        __syncthreads();
        const int ky = k + D < nblk ? k + D : -1;
        for (int qi = 0; qi < nq; ++qi) quad_pass(qi, k, nv, ky);
        if (ky >= 0) release_y(ky);
        __syncthreads();  // ring slot / d0s reuse
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int e = tid; e < nq * RPCp; e += NT) {
        const int qi = e / RPCp, li = e - qi * RPCp;
        if (li < nr) *reinterpret_cast<float4*>(A.W0 + (size_t)(i0 + li) * H + 4 * (q0 + qi)) = wsm[e];
    }
    if (pid == 0 && n > 0) {
        const float* xl = A.X + win_row(A, n - 1) * I;
        for (int i = tid; i < I; i += NT) A.x0[i] = xl[i];
    }
}

// Producer for the single-CTA chain (H <= 256): one column quad per CTA.
// (The multi-quad producer above costs ~3% at C2: an extra barrier per quad
// and a later Y release.)
template <int NT>
__device__ __forceinline__ void win_producer_v1(const WinArgs& A, float* sm) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = A.I, H = A.H, D = A.D, KS = A.KS, RPC = A.RPC;
    const int pc = (blockIdx.x - 1) / KS, ks = (blockIdx.x - 1) - pc * KS;
    const int col = 4 * pc, i0 = ks * RPC, nr = max(0, min(I, i0 + RPC) - i0);
    const int n = A.n_steps;
    const int nblk = (n + kWinS - 1) / kWinS;
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    const ProdSmem L(RPC, D);
    const int RPCp = L.RPCp, NB = L.NB;
    float* xr = sm + L.xr;
    float* red = sm + L.red;
    float4* d0s = reinterpret_cast<float4*>(sm + L.d0s);
    const bool vec = ((I & 3) == 0) && ((i0 & 3) == 0) && ((nr & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(A.X) & 15) == 0);

    float4 w[kWinMaxNR];
#pragma unroll
    for (int m = 0; m < kWinMaxNR; ++m) {
        const int li = tid + NT * m;
        w[m] = li < nr ? *reinterpret_cast<const float4*>(A.W0 + (size_t)(i0 + li) * H + col)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // X rows [i0, i0+nr) of block blk -> ring slot blk % NB (cp.async, no wait)
    auto prefetch = [&](int blk) {
        float* dst = xr + (size_t)(blk % NB) * kWinS * RPCp;
        const int s0 = blk * kWinS, nv = min(kWinS, n - s0);
        if (vec) {
            const int nq = nr >> 2;
            for (int e = tid; e < nv * nq; e += NT) {
                const int u = e / nq, q = e - u * nq;
                cp_async16(dst + u * RPCp + 4 * q, A.X + win_row(A, s0 + u) * I + i0 + 4 * q);
            }
        } else {
            for (int e = tid; e < nv * nr; e += NT) {
                const int u = e / nr, q = e - u * nr;
                cp_async4(dst + u * RPCp + q, A.X + win_row(A, s0 + u) * I + i0 + q);
            }
        }
    };
    // partial Y(blk)[u][col..col+3] over this row range, from the current registers
    auto compute_y = [&](int blk) {
        const float* xb = xr + (size_t)(blk % NB) * kWinS * RPCp;
        const int nv = min(kWinS, n - blk * kWinS);
        float acc[4 * kWinS];
#pragma unroll
        for (int e = 0; e < 4 * kWinS; ++e) acc[e] = 0.0f;
#pragma unroll
        for (int m = 0; m < kWinMaxNR; ++m) {
            const int li = tid + NT * m;
            if (li < nr) {
#pragma unroll
                for (int u = 0; u < kWinS; ++u) {
                    const float x = u < nv ? xb[u * RPCp + li] : 0.0f;
                    acc[4 * u + 0] = fmaf(x, w[m].x, acc[4 * u + 0]);
                    acc[4 * u + 1] = fmaf(x, w[m].y, acc[4 * u + 1]);
                    acc[4 * u + 2] = fmaf(x, w[m].z, acc[4 * u + 2]);
                    acc[4 * u + 3] = fmaf(x, w[m].w, acc[4 * u + 3]);
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
            for (int q = 0; q < NT / 32; ++q) y += red[q * 64 + tid];
            const int u = tid >> 2, c = tid & 3;
            if (u < nv) __stcg(A.yring + (((size_t)(blk % YR) * KS + ks) * kWinS + u) * H + col + c, y);
            // each of the two writer warps releases its own stores
            __syncwarp();
            if (lane == 0) red_release_add(A.ycnt + (blk % YR), 1u);
        }
    };

    const int npro = min(D, nblk);
    for (int blk = 0; blk <= npro && blk < nblk; ++blk) prefetch(blk);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int blk = 0; blk < npro; ++blk) {
        compute_y(blk);
        __syncthreads();  // red reuse
    }
    for (int k = 0; k < nblk; ++k) {
        const int nv = min(kWinS, n - k * kWinS);
        if (k + D + 1 < nblk) prefetch(k + D + 1);  // slot of block k-1: retired
        cp_async_commit();
        if (tid == 0) spin_geq(A.dcnt, (unsigned)(k + 1), A.error);
        __syncthreads();
        if (tid < kWinS)
            d0s[tid] = tid < nv ? __ldcg(reinterpret_cast<const float4*>(
                                      A.dring + ((size_t)(k % DR) * kWinS + tid) * H + col))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        cp_async_wait<1>();  // block k+D's rows (prefetched last iteration) have landed
        __syncthreads();
        // the S per-sample updates, reference rounding, in sample order
        const float* xb = xr + (size_t)(k % NB) * kWinS * RPCp;
#pragma unroll
        for (int m = 0; m < kWinMaxNR; ++m) {
            const int li = tid + NT * m;
            if (li < nr) {
#pragma unroll
                for (int u = 0; u < kWinS; ++u) {
                    if (u < nv) {
                        const float4 d = d0s[u];
                        const float x = xb[u * RPCp + li];
                        w[m].x = sgd_apply(w[m].x, neg_eta, d.x, x);
                        w[m].y = sgd_apply(w[m].y, neg_eta, d.y, x);
                        w[m].z = sgd_apply(w[m].z, neg_eta, d.z, x);
                        w[m].w = sgd_apply(w[m].w, neg_eta, d.w, x);
                    }
                }
            }
        }
        if (k + D < nblk) compute_y(k + D);
        __syncthreads();  // ring slot / d0s / red reuse
    }
    cp_async_wait<0>();
#pragma unroll
    for (int m = 0; m < kWinMaxNR; ++m) {
        const int li = tid + NT * m;
        if (li < nr) *reinterpret_cast<float4*>(A.W0 + (size_t)(i0 + li) * H + col) = w[m];
    }
    if (blockIdx.x == 1 && n > 0) {
        const float* xl = A.X + win_row(A, n - 1) * I;
        for (int i = tid; i < I; i += NT) A.x0[i] = xl[i];
    }
}

__device__ __forceinline__ unsigned ld_acquire_cta_u32(uint32_t saddr) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_u32(uint32_t saddr, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;\n" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(x));
    return r;
}

// ---------------------------------------------------------------------------
// Chain CTA.
// ---------------------------------------------------------------------------
template <int JPL, int CT, int NCW, bool CLU, bool DIR, bool TR>
__device__ __forceinline__ void win_chain(const WinArgs& A, float* sm, const WinSmem& L) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // CS chain CTAs (one cluster) split the hidden layer: rank r owns units
    // [h0, h0 + Hs); everything H-wide in this CTA is slice-local
    const int CS = CLU ? A.CS : 1, rank = CLU ? (int)cluster_ctarank() : 0;
    const int H = A.H, Hs = H / CS, h0 = rank * Hs;
    const int D = A.D, HP = L.HP, R = L.R, Rd = L.Rd, QW = A.QW, KS = A.KS;
    const int HQ = Hs >> 2;  // float4 per slice row
    const int C = CT > 0 ? CT : A.C;
    const int n = (int)A.n_steps;  // <= 2^18 per launch (host chunks the stream)
    const int nblk = (n + kWinS - 1) / kWinS;
    const int YR = D + 1, DR = D + 1;
    const float neg_eta = A.neg_eta;
    float* zacc = sm + L.zacc;
    float* ystage = sm + L.ystage;
    float* tstage = sm + L.tstage;
    float* coefs = sm + L.coefs;
    float* d0ring = sm + L.d0ring;
    float* pring = sm + L.pring;
    float* red = sm + L.red;
    unsigned* rowflag = reinterpret_cast<unsigned*>(sm + L.rowflag);
    float* gat = sm + L.gat;
    const uint32_t mb = smem_u32(sm + L.mbar);
    auto MB = [&](int idx) { return mb + 8u * (uint32_t)idx; };
    unsigned long long* const trace = A.trace;
#define WIN_TRACE(s_, ph)                                                                \
    do {                                                                                 \
        if (TR && trace && lane == 0 && (unsigned)((s_) - A.trace_base) < kTraceSamples)       \
            trace[((s_) - A.trace_base) * kTracePhases + (ph)] = clock64();              \
    } while (0)

    // ---- prologue: zero the rings, init the barriers
    for (int e = tid; e < R * HP; e += win_threads<NCW>()) zacc[e] = 0.0f;
    for (int e = tid; e < 2 * A.KS * kWinS * Hs; e += win_threads<NCW>()) ystage[e] = 0.0f;
    for (int e = tid; e < 2 * kWinS * kWinCP; e += win_threads<NCW>()) tstage[e] = 0.0f;
    for (int e = tid; e < L.Rdh * HP; e += win_threads<NCW>()) d0ring[e] = 0.0f;
    for (int e = tid; e < R; e += win_threads<NCW>()) rowflag[e] = 0u;
    if (tid == 0) {
        for (int r = 0; r < kWinRing; ++r) mbar_init(MB(kMbD0 + r), 32 * NCW);
        for (int r = 0; r < 2; ++r) {
            mbar_init(MB(kMbYFull + r), 32);
            mbar_init(MB(kMbYFree + r), 32 * NCW);
        }
        for (int r = 0; r < kWinBlkRing; ++r) mbar_init(MB(kMbBlk + r), 32 * NCW);
        if (CS > 1) {
            // one local arrival (with the expected bytes) + CS*C st.async completions
            mbar_init(MB(kMbXch + 0), 1);
            mbar_init(MB(kMbXch + 1), 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            if (n > 0) mbar_arrive_expect_tx(MB(kMbXch + 0), (uint32_t)(CS * C * sizeof(float)));
            if (n > 1) mbar_arrive_expect_tx(MB(kMbXch + 1), (uint32_t)(CS * C * sizeof(float)));
        }
    }
    __syncthreads();
    if (CS > 1) cluster_sync_all();  // every chain CTA initialised before remote traffic

    if (win_chain_index<NCW>(warp) >= 0) {
        // ================= the serial chain (NCW warps) =================
        // chain warp cw owns hidden units [cw*32*JPL + JPL*lane, +JPL); the
        // partial logits of the NCW warps meet in shared memory once per sample
        constexpr int CC = CT > 0 ? CT : kWinCP;
        constexpr int XS = 32 * NCW + 4;  // row stride of the transposed partials
        const int cw = win_chain_index<NCW>(warp);
        const int j0 = cw * 32 * JPL + JPL * lane;  // first owned hidden unit (slice-local)
        const bool jval = j0 < Hs;                  // Hs % 4 == 0: all JPL units valid or none
        const bool kval = lane < C;                 // lane k also owns class k (totals, b1)
        const int kr = lane & (kWinCP - 1);         // class row summed by this lane
        float w1[JPL][CC], b0r[JPL], dp1[JPL], dp2[JPL], aprev[JPL], naprev[JPL], d1p[CC];
#pragma unroll
        for (int m = 0; m < JPL; ++m) {
            const int j = j0 + m;
#pragma unroll
            for (int k = 0; k < CC; ++k) w1[m][k] = (j < Hs && k < C) ? A.W1[(size_t)(h0 + j) * C + k] : 0.0f;
            b0r[m] = j < Hs ? A.b0[h0 + j] : 0.0f;
            dp1[m] = dp2[m] = aprev[m] = naprev[m] = 0.0f;
        }
#pragma unroll
        for (int k = 0; k < CC; ++k) d1p[k] = 0.0f;
        float b1k = kval ? A.b1[lane] : 0.0f;  // every chain warp keeps an identical copy
        float zl[JPL], zkl = 0.0f, pkl = 0.0f, dkl = 0.0f;  // last sample's z0, z1, p, d1
#pragma unroll
        for (int m = 0; m < JPL; ++m) zl[m] = 0.0f;
        float* const xr = red;                                // [16][XS] partial logits
        float* const half0 = red + kWinCP * XS;                   // [2][NCW][16] per-warp class sums
        float* const zt = half0 + 2 * NCW * kWinCP + cw * kWinCP;  // this warp's logits copy
        float* const es = zt + NCW * kWinCP;                       // this warp's exponentials copy
        // prefetched operands of the next sample (raw: sums at first use)
        constexpr int kMaxKS = 2;  // the plan uses at most 2 row splits
        struct Pre {
            float zraw[JPL], yraw[kMaxKS][JPL], tn[CC];
            float c1n, c2n, town;
        };
        Pre pa, pb;
        pa.c1n = pa.c2n = pa.town = pb.c1n = pb.c2n = pb.town = 0.0f;
        auto flag_wait = [&](int s1, int s1R) {
            if (s1 < 3) return;  // rows 0..2: the chain applies every correction itself
            const uint32_t fa = smem_u32(rowflag + s1R);
            const unsigned want = (unsigned)(s1 + 1);
            if (ld_acquire_cta_u32(fa) != want) {
                const unsigned long long t0 = globaltimer_ns();
                while (ld_acquire_cta_u32(fa) != want) {
                    if (globaltimer_ns() - t0 > 5000000000ull) {
                        atomicExch(A.error, 4);
                        __trap();
                    }
                }
            }
        };
        // s1R = s1 % R, s1Rd = s1 % Rd (ring slots), kept incrementally
        auto fetch_row = [&](int s1, int s1R, int s1Rd, Pre& dst) {
            float(&zraw)[JPL] = dst.zraw;
            float(&yraw)[kMaxKS][JPL] = dst.yraw;
            float(&tn)[CC] = dst.tn;
            float& c1n = dst.c1n;
            float& c2n = dst.c2n;
            float& town = dst.town;
            const int b1 = s1 >> 4, u1 = s1 & (kWinS - 1), st1 = b1 & 1;
            if (u1 == 0) mbar_wait_cta(MB(kMbYFull + st1), (uint32_t)((b1 >> 1) & 1), A.error);
            vld<JPL>(zacc + s1R * HP + j0, zraw);
            const float* yr = ystage + ((size_t)st1 * KS * kWinS + u1) * Hs + j0;
#pragma unroll
            for (int p = 0; p < kMaxKS; ++p) {
                if (jval && p < KS)
                    vld<JPL>(yr + p * kWinS * Hs, yraw[p]);
                else
#pragma unroll
                    for (int m = 0; m < JPL; ++m) yraw[p][m] = 0.0f;
            }
            const float* tr = tstage + (st1 * kWinS + u1) * kWinCP;
#pragma unroll
            for (int k4 = 0; k4 < (CC + 3) / 4; ++k4) {
                const float4 t4 = reinterpret_cast<const float4*>(tr)[k4];
                if (4 * k4 + 0 < CC) tn[4 * k4 + 0] = t4.x;
                if (4 * k4 + 1 < CC) tn[4 * k4 + 1] = t4.y;
                if (4 * k4 + 2 < CC) tn[4 * k4 + 2] = t4.z;
                if (4 * k4 + 3 < CC) tn[4 * k4 + 3] = t4.w;
            }
            town = kval ? tr[lane] : 0.0f;
            const int p1 = s1Rd == 0 ? Rd - 1 : s1Rd - 1, p2 = p1 == 0 ? Rd - 1 : p1 - 1;
            c1n = s1 >= 1 ? coefs[p1 * QW + 0] : 0.0f;  // c(s1, 1) = coef[s1-1][0]
            c2n = s1 >= 2 ? coefs[p2 * QW + 1] : 0.0f;  // c(s1, 2) = coef[s1-2][1]
        };
        // cluster exchange of this CTA's slice partial logits (lanes k < C hold
        // class k): st.async to every peer (completing the peer's exchange
        // barrier), wait for all CS, sum in rank order -- identical logits in
        // every chain CTA.  The pushing warp re-arms the barrier for sample
        // s+2: no peer sends s+2 before it holds this CTA's s+1 partials, which
        // are pushed after this point.
        auto xchg = [&](int s, float part, bool push) {
            const int par = s & 1;
            const uint32_t slot = smem_u32(gat + (par * kWinMaxCS + rank) * kWinCP + lane);
            const uint32_t xb = MB(kMbXch + par);
            if (push && kval)
                for (int p = 0; p < CS; ++p) st_async_f32(mapa_shared(slot, p), part, mapa_shared(xb, p));
            {
                const unsigned long long t0 = globaltimer_ns();
                while (!mbar_try_wait(xb, (uint32_t)((s >> 1) & 1))) {
                    if (globaltimer_ns() - t0 > 5000000000ull) {
                        atomicExch(A.error, 5);
                        __trap();
                    }
                }
            }
            if (push && lane == 0 && s + 2 < n) mbar_arrive_expect_tx(xb, (uint32_t)(CS * C * sizeof(float)));
            const float* g = gat + par * kWinMaxCS * kWinCP + kr;
            float tot = g[0];
            for (int p = 1; p < CS; ++p) tot += g[p * kWinCP];
            return tot;
        };
        if (n > 0) fetch_row(0, 0, 0, pa);
        int sR = 0, sRd = 0;      // s % R, s % Rd
        int nR = 1 % R, nRd = 1;  // (s+1) % R, (s+1) % Rd
        auto body = [&](const int s, Pre& cur, Pre& nxt) {
            const int b = s >> 4, u = s & (kWinS - 1), st = b & 1;
            WIN_TRACE(s, 0);
            // -- z(s) = Y + window + c1 d0(s-1) + c2 d0(s-2) + b0;  tanh.
            //    The deferred W1 update of s-1 fills the tanh latency.
            float z[JPL], a[JPL], t[CC];
            const float tow = cur.town;
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                const float y = cur.zraw[m] + (cur.yraw[0][m] + cur.yraw[1][m]);
                z[m] = fmaf(cur.c1n, dp1[m], fmaf(cur.c2n, dp2[m], y)) + b0r[m];
                a[m] = tanhf(z[m]);
            }
#pragma unroll
            for (int k = 0; k < CC; ++k) t[k] = cur.tn[k];
            WIN_TRACE(s, 14);
            // row s+1 was flagged by its helper ~2 samples ago: fetch it now so
            // the shared-memory latency hides under this sample's chain
            if (s + 1 < n) {
                flag_wait(s + 1, nR);
                fetch_row(s + 1, nR, nRd, nxt);
            }
            WIN_TRACE(s, 15);
            // FAST numerics: the W1 update as one FMA, w + d1 (-eta a)
#pragma unroll
            for (int m = 0; m < JPL; ++m)
#pragma unroll
                for (int k = 0; k < CC; ++k) w1[m][k] = fmaf(d1p[k], naprev[m], w1[m][k]);
            WIN_TRACE(s, 1);
            // -- partial logits -> shared memory (transposed); each warp sums its
            //    own 32 columns per class, then one barrier joins the NCW warps
#pragma unroll
            for (int k = 0; k < CC; ++k) {
                float acc = 0.0f;
#pragma unroll
                for (int m = 0; m < JPL; ++m) acc = fmaf(a[m], w1[m][k], acc);
                xr[k * XS + cw * 32 + lane] = acc;
            }
            __syncwarp();
            float zown1 = 0.0f;
            {
                const float4* col = reinterpret_cast<const float4*>(xr + kr * XS + cw * 32);
                float4 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = col[q];
                float t8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) t8[q] = (v[q].x + v[q].y) + (v[q].z + v[q].w);
                const float hs = ((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]));
                // halves are double-buffered by sample parity: a warp can run one
                // sample ahead of its peer past the barrier, never two
                float* const half = half0 + (s & 1) * NCW * kWinCP;
                if (NCW > 1) {
                    if (kval) half[cw * kWinCP + lane] = hs;
                } else if (CS > 1) {
                    zown1 = sadd(xchg(s, hs, true), b1k);
                    if (kval) zt[lane] = zown1;
                } else {
                    zown1 = sadd(hs, b1k);
                    if (kval) zt[lane] = zown1;
                }
            }
            float zown = zown1;
            if (NCW > 1) {
                named_sync(1, 32 * NCW);
                const float* const half = half0 + (s & 1) * NCW * kWinCP;
                float hsum = half[kr];
#pragma unroll
                for (int c = 1; c < NCW; ++c) hsum += half[c * kWinCP + kr];
                if (CS > 1) hsum = xchg(s, hsum, cw == 0);  // chain warp 0 pushes, all wait
                zown = sadd(hsum, b1k);
                if (kval) zt[lane] = zown;
            }
            __syncwarp();
            WIN_TRACE(s, 2);
            // -- softmax: the exact max over the C logits in one warp reduction
            //    (redux.sync.max.f32); lane k computes exp(z_k - max) once and
            //    shares it through shared memory
            constexpr int CV = (CC + 3) / 4;  // float4 loads of a class vector
            float mx;
            asm("redux.sync.max.f32 %0, %1, 0xffffffff;\n" : "=f"(mx) : "f"(kval ? zown : -INFINITY));
            const float eown = expf(zown - mx);
            if (kval) es[lane] = eown;
            __syncwarp();
            float ek[4 * CV];
#pragma unroll
            for (int k4 = 0; k4 < CV; ++k4) {
                const float4 v = reinterpret_cast<const float4*>(es)[k4];
                ek[4 * k4 + 0] = v.x;
                ek[4 * k4 + 1] = v.y;
                ek[4 * k4 + 2] = v.z;
                ek[4 * k4 + 3] = v.w;
            }
#pragma unroll
            for (int k = 0; k < 4 * CV; ++k)
                if (k >= CC || (CT == 0 && k >= C)) ek[k] = 0.0f;
            // tree sum (fixed order)
            float sp[4 * CV];
#pragma unroll
            for (int k = 0; k < 4 * CV; ++k) sp[k] = ek[k];
#pragma unroll
            for (int wdt = 1; wdt < 4 * CV; wdt <<= 1)
#pragma unroll
                for (int k = 0; k + wdt < 4 * CV; k += 2 * wdt) sp[k] += sp[k + wdt];
            const float inv = rcp_approx(sp[0]);
            float d1[CC];
#pragma unroll
            for (int k = 0; k < CC; ++k) d1[k] = k < C ? fmaf(ek[k], inv, -t[k]) : 0.0f;  // p - t
            // d0 = (1 - a^2) * (W1 d1) with the pre-update W1 (two half-chains:
            // the dependent FMA latency is on the critical path)
            float d0v[JPL];
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
                for (int k = 0; k < CC / 2; ++k) acc0 = fmaf(d1[k], w1[m][k], acc0);
#pragma unroll
                for (int k = CC / 2; k < CC; ++k) acc1 = fmaf(d1[k], w1[m][k], acc1);
                d0v[m] = fmaf(-a[m], a[m], 1.0f) * (acc0 + acc1);  // (1 - a^2) W1 d1
            }
            WIN_TRACE(s, 3);
            if constexpr (DIR) {
                // helpers read the short smem ring; producers read the L2 ring
                // (the publisher releases it per block, cumulatively)
                vst<JPL>(d0ring + (s & (kWinS - 1)) * HP + j0, d0v);
                if (jval) vst<JPL>(A.dring + ((size_t)(b % (D + 1)) * kWinS + u) * H + h0 + j0, d0v);
            } else {
                vst<JPL>(d0ring + sRd * HP + j0, d0v);
            }
            mbar_arrive_cta(MB(kMbD0 + (s & (kWinRing - 1))));
            WIN_TRACE(s, 4);
            // -- off the chain: p and d1 of the lane's own class, stats, biases
#pragma unroll
            for (int k = 0; k < CC; ++k) d1p[k] = d1[k];
            const float pk = eown * inv;
            const float dk = kval ? ssub(pk, tow) : 0.0f;
            if (cw == 0 && rank == 0 && kval) pring[sRd * kWinCP + lane] = pk;
            b1k = fmaf(neg_eta, dk, b1k);
            zkl = zown;
            pkl = pk;
            dkl = dk;
            if (u == kWinS - 1 || s == n - 1) {
                mbar_arrive_cta(MB(kMbBlk + b % kWinBlkRing));
                mbar_arrive_cta(MB(kMbYFree + st));
            }
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                b0r[m] = fmaf(neg_eta, d0v[m], b0r[m]);
                dp2[m] = dp1[m];
                dp1[m] = d0v[m];
                aprev[m] = a[m];
                naprev[m] = neg_eta * a[m];
                zl[m] = z[m];
            }
            WIN_TRACE(s, 5);
            sR = nR;
            sRd = nRd;
            if (++nR == R) nR = 0;
            if (++nRd == Rd) nRd = 0;
            WIN_TRACE(s, 6);
        };
        // unrolled by two: the prefetch of row s+1 lands in the other register
        // set (no copies of the prefetched row between samples)
        for (int s = 0; s < n; s += 2) {
            body(s, pa, pb);
            if (s + 1 < n) body(s + 1, pb, pa);
        }
        if (n > 0) {
            // the last sample's W1 update (deferred in the loop)
#pragma unroll
            for (int m = 0; m < JPL; ++m)
#pragma unroll
                for (int k = 0; k < CC; ++k) w1[m][k] = fmaf(d1p[k], naprev[m], w1[m][k]);
#pragma unroll
            for (int m = 0; m < JPL; ++m) {
                const int j = j0 + m;
                if (j < Hs) {
                    const int jg = h0 + j;
#pragma unroll
                    for (int k = 0; k < CC; ++k)
                        if (k < C) A.W1[(size_t)jg * C + k] = w1[m][k];
                    A.b0[jg] = b0r[m];
                    A.z0[jg] = zl[m];
                    A.a0[jg] = aprev[m];
                    A.d0[jg] = dp1[m];
                    A.db0[jg] = smul(neg_eta, dp1[m]);
                    A.x1[jg] = aprev[m];
                }
            }
            if (cw == 0 && rank == 0 && kval) {
                A.b1[lane] = b1k;
                A.z1[lane] = zkl;
                A.a1[lane] = pkl;
                A.d1[lane] = dkl;
                A.db1[lane] = smul(neg_eta, dkl);
            }
        }
    } else if (warp == win_loader_warp<NCW>()) {
        // ================= loader: Y(b), targets, coefficient rows =================
        // Forward band rows of block b (its own sources) go to ring slots
        // s % Rd with Y(b): block b-D-1's slots, long retired.
        constexpr int kCoefMax = kWinS * kWinMaxD * kWinS / 4 / 32;  // float4 per lane
        const int QW4 = QW >> 2;
        auto coef_load = [&](int blk, float4* v) {
            const int r0 = blk * kWinS, rows = max(0, min(kWinS, n - r0));
#pragma unroll
            for (int q = 0; q < kCoefMax; ++q) {
                const int e = lane + 32 * q;
                if (e < rows * QW4) {
                    const int u = e / QW4, c = e - u * QW4;
                    v[q] = __ldg(reinterpret_cast<const float4*>(A.coef + (size_t)(r0 + u) * QW) + c);
                }
            }
        };
        auto coef_store = [&](int blk, const float4* v) {
            const int r0 = blk * kWinS, rows = max(0, min(kWinS, n - r0));
#pragma unroll
            for (int q = 0; q < kCoefMax; ++q) {
                const int e = lane + 32 * q;
                if (e < rows * QW4) {
                    const int u = e / QW4, c = e - u * QW4;
                    reinterpret_cast<float4*>(coefs + ((r0 + u) % Rd) * QW)[c] = v[q];
                }
            }
        };
        for (int b = 0; b < nblk; ++b) {
            const int st = b & 1;
            const int s0 = b * kWinS;
            const int nv = min(kWinS, n - s0);
            // independent of the producers: rows, targets, coefficient rows
            const long long myrow = lane < nv ? win_row(A, s0 + lane) : 0;
            float4 cv[kCoefMax];
            coef_load(b, cv);
            float tv[kWinS * kWinCP / 32];
#pragma unroll
            for (int q = 0; q < kWinS * kWinCP / 32; ++q) {
                const int e = lane + 32 * q, u = e / kWinCP, k = e % kWinCP;
                const long long r = __shfl_sync(0xffffffffu, myrow, u);
                tv[q] = (u < nv && k < C) ? __ldg(A.T + r * C + k) : 0.0f;
            }
            WIN_TRACE(s0, 8);
            if (b >= 2) mbar_wait_cta(MB(kMbYFree + st), (uint32_t)(((b - 2) >> 1) & 1), A.error);
            spin_geq(A.ycnt + (b % YR), (unsigned)(2 * A.P * (b / YR + 1)), A.error);  // 2 writer warps per producer
            WIN_TRACE(s0, 9);
            coef_store(b, cv);
            // Y(b): the KS partial slabs of this CTA's slice by TMA bulk copy
            // (whole rows at once when the slice is the full layer), completing
            // yfull's transaction count
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic writes -> async proxy
                const uint32_t mbar = MB(kMbYFull + st);
                mbar_arrive_expect_tx(mbar, (uint32_t)(KS * nv * Hs * sizeof(float)));
                for (int p = 0; p < KS; ++p) {
                    const float* src = A.yring + (((size_t)(b % YR) * KS + p) * kWinS) * H + h0;
                    float* dst = ystage + ((size_t)st * KS + p) * kWinS * Hs;
                    const int nrow = CS == 1 ? 1 : nv;
                    const uint32_t bytes = (uint32_t)((CS == 1 ? nv * H : Hs) * sizeof(float));
                    for (int u = 0; u < nrow; ++u)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                smem_u32(dst + (size_t)u * Hs)),
                            "l"(src + (size_t)u * H), "r"(bytes), "r"(mbar)
                            : "memory");
                }
            }
#pragma unroll
            for (int q = 0; q < kWinS * kWinCP / 32; ++q) tstage[st * kWinS * kWinCP + lane + 32 * q] = tv[q];
            if (lane != 0) mbar_arrive_cta(MB(kMbYFull + st));  // lane 0 arrived with expect_tx
            WIN_TRACE(s0, 10);
        }
    } else if (warp == win_pub_warp<NCW>()) {
        // ================= publisher: d0 blocks to L2, loss/accuracy =================
        double loss_acc = (lane == 0 && A.loss_sum) ? *A.loss_sum : 0.0;
        unsigned long long correct_acc = 0;
        const bool stats = (A.loss_sum || A.correct) && rank == 0;
        for (int k = 0; k < nblk; ++k) {
            const int s0 = k * kWinS;
            const int nv = min(kWinS, n - s0);
            // target row of sample s0+lane (independent of the chain)
            const long long myrow = (stats && lane < nv) ? win_row(A, s0 + lane) : 0;
            mbar_wait_cta(MB(kMbBlk + k % kWinBlkRing), (uint32_t)((k / kWinBlkRing) & 1), A.error);
            WIN_TRACE(s0, 11);
            // this CTA's slice of the block's d0 rows (dring rows are H wide);
            // multi-warp cluster chains wrote them directly (the fence below makes
            // the chain warps' stores, ordered before blkdone, visible with the
            // release)
            if constexpr (!DIR) {
                float* dst = A.dring + (size_t)(k % DR) * kWinS * H + h0;
                for (int e = lane; e < nv * HQ; e += 32) {
                    const int u = e / HQ, q = e - u * HQ;
                    __stcg(reinterpret_cast<float4*>(dst + (size_t)u * H) + q,
                           reinterpret_cast<const float4*>(d0ring + ((s0 + u) % Rd) * HP)[q]);
                }
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) red_release_add(A.dcnt, 1u);
            WIN_TRACE(s0 + 1, 11);
            if (stats) {
                // lane u: loss / hit of sample s0+u (network.cpp:165-168), then
                // lane 0 accumulates in sample order
                float loss = 0.0f;
                unsigned hit = 0;
                if (lane < nv) {
                    const float* tc = A.T + myrow * C;
                    const float* pl = pring + ((s0 + lane) % Rd) * kWinCP;
                    int bp = 0, btg = 0;
                    float tb = __ldg(tc);
                    for (int o = 0; o < C; ++o) {
                        const float to = __ldg(tc + o);
                        if (to != 0.0f) {
                            const float q = pl[o] < 1e-12f ? 1e-12f : pl[o];
                            loss = ssub(loss, smul(to, logf(q)));
                        }
                        if (pl[o] > pl[bp]) bp = o;
                        if (to > tb) {
                            btg = o;
                            tb = to;
                        }
                    }
                    hit = bp == btg;
                }
                for (int u = 0; u < nv; ++u) {
                    const float lu = __shfl_sync(0xffffffffu, loss, u);
                    loss_acc = __dadd_rn(loss_acc, (double)lu);
                }
                correct_acc += __popc(__ballot_sync(0xffffffffu, hit != 0));
            }
            WIN_TRACE(s0 + 2, 11);
        }
        if (lane == 0 && rank == 0) {
            if (A.loss_sum) *A.loss_sum = loss_acc;
            if (A.correct) *A.correct += correct_acc;
        }
    } else if (win_helper_index<NCW>(warp) >= 0) {
        // ================= helpers: window corrections =================
        // d0(s) goes to every pending row r in [s+3, last] owned by this warp
        // (r = w mod NH): z(r) += c(r, r-s) d0(s), c from the forward band row
        // of source s.  Rows are visited in ascending order, so an owned row
        // s+3 (the next one the chain fetches) is flagged first.
        const int w = win_helper_index<NCW>(warp);
        int sR = 0, sRd = 0;  // s % R, s % Rd
        for (int s = 0; s < n; ++s) {
            const int b = s >> 4;
            const int last = min(n - 1, (b + D) * kWinS - 1);
            const int f0 = s + 3;
            const int first = f0 + ((w - (f0 & (kWinHelpers - 1))) & (kWinHelpers - 1));
            mbar_wait_cta(MB(kMbD0 + (s & (kWinRing - 1))), (uint32_t)((s >> 4) & 1), A.error);
            if ((s & (kWinHelpers - 1)) == w) WIN_TRACE(s, 12);
            const float4* dv =
                reinterpret_cast<const float4*>(d0ring + (DIR ? (s & (kWinS - 1)) : sRd) * HP);
            const float* cs = coefs + sRd * QW - s - 1;  // cs[r] = c(r, r-s)
            // this lane's d0 quads, once per sample
            constexpr int NQH = JPL * NCW / 4;  // float4 per lane per row (HP = 32 JPL NCW)
            float4 dq[NQH];
#pragma unroll
            for (int i = 0; i < NQH; ++i) {
                const int q = lane + 32 * i;
                dq[i] = q < HQ ? dv[q] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            auto upd = [&](float4* zr, float c) {
#pragma unroll
                for (int i = 0; i < NQH; ++i) {
                    const int q = lane + 32 * i;
                    if (q < HQ) {
                        float4 z = zr[q];
                        z.x = fmaf(c, dq[i].x, z.x);
                        z.y = fmaf(c, dq[i].y, z.y);
                        z.z = fmaf(c, dq[i].z, z.z);
                        z.w = fmaf(c, dq[i].w, z.w);
                        zr[q] = z;
                    }
                }
            };
            int slot = sR + (first - s);
            if (slot >= R) slot -= R;
            int r = first;
            if (r == f0 && r <= last) {  // the next row the chain fetches: flag it first
                upd(reinterpret_cast<float4*>(zacc + slot * HP), cs[r]);
                __syncwarp();
                if (lane == 0) st_release_cta_u32(smem_u32(rowflag + slot), (unsigned)(f0 + 1));
                WIN_TRACE(f0, 7);
                r += kWinHelpers;
                slot += kWinHelpers;
                if (slot >= R) slot -= R;
            }
            // the rest, 4 independent rows per batch
            for (; r <= last; r += 4 * kWinHelpers) {
                int sl[4];
                float c[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    sl[k] = slot;
                    c[k] = r + k * kWinHelpers <= last ? cs[r + k * kWinHelpers] : 0.0f;
                    slot += kWinHelpers;
                    if (slot >= R) slot -= R;
                }
#pragma unroll
                for (int i = 0; i < NQH; ++i) {
                    const int q = lane + 32 * i;
                    if (q < HQ) {
                        float4 z[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (r + k * kWinHelpers <= last) z[k] = reinterpret_cast<const float4*>(zacc + sl[k] * HP)[q];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (r + k * kWinHelpers <= last) {
                                z[k].x = fmaf(c[k], dq[i].x, z[k].x);
                                z[k].y = fmaf(c[k], dq[i].y, z[k].y);
                                z[k].z = fmaf(c[k], dq[i].z, z[k].z);
                                z[k].w = fmaf(c[k], dq[i].w, z[k].w);
                                reinterpret_cast<float4*>(zacc + sl[k] * HP)[q] = z[k];
                            }
                        }
                    }
                }
            }
            // the chain read row s before publishing d0(s): its slot now
            // belongs to row s + R (first corrected by block(s)+1's d0)
            if ((s & (kWinHelpers - 1)) == w) {
                float4* zr = reinterpret_cast<float4*>(zacc + sR * HP);
                for (int q = lane; q < HQ; q += 32) zr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if ((s & (kWinHelpers - 1)) == w) WIN_TRACE(s, 13);
            if (++sR == R) sR = 0;
            if (++sRd == Rd) sRd = 0;
        }
    }
#undef WIN_TRACE
    if (CS > 1) cluster_sync_all();  // no chain CTA exits while a peer may still address it
}

// JPL hidden units per chain lane, CT classes (0 = runtime <= 16), NCW chain
// warps, CLU: the chain is split over a cluster of A.CS CTAs (else one CTA),
// MQ/NR: max column quads per producer CTA / W0 rows per producer thread;
// TR: per-phase clock64 trace of the chain CTA (diagnostics build only)
template <int JPL, int CT, int NCW, bool CLU = false, int MQ = 1, int NR = kWinMaxNR, bool TR = false>
__global__ void __launch_bounds__(win_threads<NCW>(), 1) k_sgd_window(WinArgs A) {
    extern __shared__ __align__(16) float sm[];
    if ((int)blockIdx.x < (CLU ? A.CS : 1))
        // DIR: d0 straight to the L2 ring (multi-warp or 16-CTA cluster chains,
        // where it measured faster and saves shared memory)
        win_chain<JPL, CT, NCW, CLU, CLU && (NCW >= 2 || MQ >= 8), TR>(
            A, sm, WinSmem(32 * JPL * NCW, A.D, A.KS, A.H / (CLU ? A.CS : 1), NCW, CLU && (NCW >= 2 || MQ >= 8)));
    else if constexpr (!CLU)
        win_producer_v1<win_threads<NCW>()>(A, sm);
    else if constexpr (MQ == kWinSmemQPC)
        win_producer_smem<win_threads<NCW>(), NR>(A, sm);
    else
        win_producer<win_threads<NCW>(), MQ, NR>(A, sm);
}

}  // namespace lane_b200
