// gemm_tcp.cuh -- the persistent form of the tcgen05 3xTF32 GEMM (gemm_tc.cuh)
// for the shapes a one-tile-per-CTA launch serves badly: the mini-batch GEMMs
// whose 128x128 tiles are too few for 148 SMs (M = batch = 256: 64 tiles) and
// the short-K wgrads (K = batch: 8 K blocks per tile, where fill/drain and the
// epilogue dominate).
//
// One CTA per SM loops over work units.  A work unit is a contiguous range of
// K blocks of one 128x128 output tile:
//   * data parallel (tiles >= 2 waves): CTA c takes whole tiles c, c + grid, ...
//     in a grouped raster (GROUP tile rows at a time, for L2 reuse of B);
//   * stream-K (fewer tiles): the tiles x K-blocks iteration space is cut into
//     grid equal contiguous ranges, one per CTA (grid <= #SMs, one CTA per SM);
//     a tile covered by several ranges is finished by its piece 0 (the one
//     holding K block 0, the LAST unit of its CTA's range), which waits for
//     the later pieces' raw partials -- they open their CTAs' ranges, so they
//     are normally long published -- and sums them in piece (= K) order,
//     deterministically, before the fused epilogue.  The wait is bounded
//     (5 s, then trap: a failure, never a hang).
// Warp roles (448 threads):
//   warp 0      TMA producer: runs ahead across units through the 4-stage ring
//   warp 1      MMA issuer: 3xTF32 MMAs (A from TMEM) into one of TWO TMEM
//               accumulators, so a unit's MMAs overlap the previous unit's
//               epilogue
//   warps 2..9  split pass (A, A_lo -> TMEM; B_lo -> smem), as in gemm_tc.cuh
//   warps 10..13 epilogue: TMEM -> registers -> fused epilogue -> global
// TMEM (512 columns): accumulators [0,128) and [128,256), then per stage 64
// columns of A and A_lo.
// Epilogues: those of gemm_tc.cuh plus UPDATE, the wgrad fused with the
// SGD/momentum step of minibatch.cuh (k_momentum_update_all's exact operation
// sequence per element: G = acc * (1/B); V = mu V + (-eta) G; W += V).
#pragma once

#include "gemm_tc.cuh"

namespace lane_b200 {

constexpr int kTpStages = 4;      // ring stages (TMEM: 2 accumulators + 4 x 64 A / A_lo columns)
constexpr int kTpSplitWarps = 8;
constexpr int kTpEpiWarps = 4;
constexpr int kTpThreads = 32 * (2 + kTpSplitWarps + kTpEpiWarps);
constexpr int kTpBTile = kTcBN * kTcBK * 4;           // 128 x 32 fp32
// a stage: A (TMA), B (TMA); B_lo overwrites A once every split warp has
// read its A rows into registers (A goes on to TMEM), so a stage is 32 KB
// and the UPDATE kernel keeps 4 stages next to its W / V slots
constexpr int kTpStage = kTcTile + kTpBTile;
constexpr int kTpAcc = 2;                             // TMEM accumulators
constexpr int kTpTileElems = kTcBM * kTcBN;
constexpr int kTpUpdCols = 16;                        // columns per W / V chunk
constexpr int kTpUpdChunk = kTcBM * kTpUpdCols * 4;   // one 128 x 16 fp32 chunk of W or V (64B swizzle)

// UPDATE: each epilogue warp streams W and V through 6 sub-chunk slots with
// loads 5 chunks ahead, and the ring keeps 4 MMA stages.  (The first version
// used 128 x 32 chunks: 4 slots left room for 2 ring stages only, and the
// K-block ring -- TMA latency + split + MMA per stage -- bound the kernel: 93 us
// for C3's 4096 x 4096 x 256 wgrad + update.)
constexpr int kTpUpdSlots = 6;
template <int E>
struct TpCfg {
    static constexpr bool kUpd = E == 4;                    // TpEpi::UPDATE
    static constexpr int kStages = kTpStages;
    static constexpr size_t kRing = (size_t)kStages * kTpStage;
    static constexpr size_t kEpi = kUpd ? kTpUpdSlots * 2 * kTpUpdChunk : 0;  // slots x (W, V)
    static constexpr size_t kSmem = kRing + kEpi + 1024 + 512;
};

enum class TpEpi : int { STORE = 0, BIAS = 1, BIAS_TANH = 2, TANH_GRAD = 3, UPDATE = 4 };

struct TpArgs {
    int M, N, K;
    int tiles_m, tiles_n, kbs;  // output tiles along M / N; K blocks per tile
    int sk;                     // 1: stream-K ranges of `per` K blocks; 0: whole tiles
    int per;                    // stream-K: K-block iterations per CTA
    int group;                  // raster: tile rows per group (data parallel)
    int max_pieces;             // stream-K: pieces per tile at most (partials layout)
    float* C;                   // M x N row-major
    float* C2;                  // BIAS_TANH: tanh(C)
    const float* bias;          // BIAS*: per column
    const float* aux;           // TANH_GRAD: activations (M x N)
    float* part;                // stream-K partial tiles [tile][piece][128 x 128]
    int* counters;              // stream-K arrivals per tile (zero between launches)
    float* W;                   // UPDATE: weights (M x N), updated in place
    float* V;                   // UPDATE: velocities / delta_weights
    float inv_b, neg_eta, mu;   // UPDATE
};

struct TpUnit {
    int tile, kb0, kb1, piece, npieces;
};

// The unit sequence of this CTA (identical in every role).  `it` is the
// role's cursor: data parallel -> the unit count so far; stream-K -> the next
// iteration of the CTA's range.
__device__ __forceinline__ bool tp_next(const TpArgs& a, long long& it, TpUnit& u) {
    const long long tiles = (long long)a.tiles_m * a.tiles_n;
    if (!a.sk) {
        const long long t = (long long)blockIdx.x + it * gridDim.x;
        if (t >= tiles) return false;
        ++it;
        u.tile = (int)t;
        u.kb0 = 0;
        u.kb1 = a.kbs;
        u.piece = 0;
        u.npieces = 1;
        return true;
    }
    const long long total = tiles * a.kbs;
    const long long beg = (long long)blockIdx.x * a.per;
    const long long end = min(total, beg + a.per);
    const long long t = beg + it;
    if (t >= end) return false;
    u.tile = (int)(t / a.kbs);
    u.kb0 = (int)(t - (long long)u.tile * a.kbs);
    const long long tile_end = (long long)(u.tile + 1) * a.kbs;
    u.kb1 = (int)(min(end, tile_end) - (long long)u.tile * a.kbs);
    it += u.kb1 - u.kb0;
    const long long first = ((long long)u.tile * a.kbs) / a.per;
    const long long last = (tile_end - 1) / a.per;
    u.piece = (int)(blockIdx.x - first);
    u.npieces = (int)(last - first + 1);
    return true;
}

// tile -> (m block, n block): grouped raster, `group` tile rows per group
__device__ __forceinline__ void tp_tile_mn(const TpArgs& a, int tile, int& mt, int& nt) {
    const int per_group = a.group * a.tiles_n;
    const int g = tile / per_group;
    const int first = g * a.group;
    const int gm = min(a.tiles_m - first, a.group);
    const int r = tile - g * per_group;
    mt = first + r % gm;
    nt = r / gm;
}

template <TpEpi E, int NV>
__device__ __forceinline__ void tp_epi_store(const TpArgs& a, int m, int n0, const float (&v)[NV]) {
    // one row segment [n0, n0 + NV) of row m (m < M checked by the caller)
    if (n0 + NV <= a.N && (a.N & 3) == 0) {
#pragma unroll
        for (int q = 0; q < NV / 4; ++q) {
            const int n = n0 + 4 * q;
            const size_t idx = (size_t)m * a.N + n;
            float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            if constexpr (E == TpEpi::UPDATE) {
                // k_momentum_update_all, element by element
                float4 w = *reinterpret_cast<const float4*>(a.W + idx);
                float4 vv = a.mu == 0.0f ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(a.V + idx);
                float* xp = &x.x;
                float* wp = &w.x;
                float* vp = &vv.x;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float g = smul(xp[i], a.inv_b);
                    xp[i] = g;
                    const float step = smul(a.neg_eta, g);
                    vp[i] = a.mu == 0.0f ? step : sadd(smul(a.mu, vp[i]), step);
                    wp[i] = sadd(wp[i], vp[i]);
                }
                *reinterpret_cast<float4*>(a.C + idx) = x;
                *reinterpret_cast<float4*>(a.V + idx) = vv;
                *reinterpret_cast<float4*>(a.W + idx) = w;
            } else {
                TcArgs t{a.M, a.N, a.K, 0, nullptr, a.C, a.C2, a.bias, a.aux};
                float4 th;
                x = tc_epi4<(TcEpi)E>(t, m, n, x, &th);
                *reinterpret_cast<float4*>(a.C + idx) = x;
                if constexpr (E == TpEpi::BIAS_TANH) *reinterpret_cast<float4*>(a.C2 + idx) = th;
            }
        }
    } else {
        for (int q = 0; q < NV; ++q) {
            const int n = n0 + q;
            if (n >= a.N) break;
            const size_t idx = (size_t)m * a.N + n;
            float x = v[q];
            if constexpr (E == TpEpi::UPDATE) {
                const float g = smul(x, a.inv_b);
                const float step = smul(a.neg_eta, g);
                const float vv = a.mu == 0.0f ? step : sadd(smul(a.mu, a.V[idx]), step);
                a.C[idx] = g;
                a.V[idx] = vv;
                a.W[idx] = sadd(a.W[idx], vv);
            } else {
                if constexpr (E == TpEpi::BIAS || E == TpEpi::BIAS_TANH) x = sadd(x, a.bias[n]);
                if constexpr (E == TpEpi::TANH_GRAD) x = tanh_grad(a.aux[idx], x);
                a.C[idx] = x;
                if constexpr (E == TpEpi::BIAS_TANH) a.C2[idx] = tanhf(x);
            }
        }
    }
}

__device__ __forceinline__ void tp_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
}

__device__ __forceinline__ void tp_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

__device__ __forceinline__ unsigned long long tp_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

__device__ __forceinline__ int tp_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void tp_epi_bar() {
    // the 4 epilogue warps only (named barrier 1)
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kTpEpiWarps) : "memory");
}

// TMA store of one 2-D box from shared memory (bulk group)
__device__ __forceinline__ void tp_tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}

template <bool A_MN, bool B_MN, TpEpi E>
__global__ void __launch_bounds__(kTpThreads, 1)
    k_gemm_tcp(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmV, TpArgs args) {
    using Cfg = TpCfg<(int)E>;
    constexpr int kTpStages = Cfg::kStages;
    extern __shared__ uint8_t tp_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tp_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* epi_buf = smem + Cfg::kRing;  // UPDATE: slot k -> W chunk at 2k, V chunk at 2k+1
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kRing + Cfg::kEpi);
    // bars: full[S], conv[S], empty[S], acc_full[2], acc_empty[2]; then the TMEM address, the last-arriver flag
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 60);  // after up to 40 barriers
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = tc_smem(smem);
    auto full = [&](int s) { return tc_smem(bars + s); };
    auto conv = [&](int s) { return tc_smem(bars + kTpStages + s); };
    auto empty = [&](int s) { return tc_smem(bars + 2 * kTpStages + s); };
    auto acc_full = [&](int b) { return tc_smem(bars + 3 * kTpStages + b); };
    auto acc_empty = [&](int b) { return tc_smem(bars + 3 * kTpStages + 2 + b); };
    // UPDATE: W / V slot k of epilogue warp (row quarter) q
    auto epi_full = [&](int q, int k) { return tc_smem(bars + 3 * kTpStages + 4 + q * kTpUpdSlots + k); };
    auto tileA = [&](int s) { return sbase + (uint32_t)(s * kTpStage); };
    auto tileB = [&](int s) { return sbase + (uint32_t)(s * kTpStage + kTcTile); };
    auto tileBlo = [&](int s) { return sbase + (uint32_t)(s * kTpStage); };  // over A, after the split

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTpStages; ++s) {
            tc_mbar_init(full(s), 1);
            tc_mbar_init(conv(s), kTpSplitWarps);
            tc_mbar_init(empty(s), 1);
        }
        for (int b = 0; b < kTpAcc; ++b) {
            tc_mbar_init(acc_full(b), 1);
            tc_mbar_init(acc_empty(b), kTpEpiWarps);
        }
        if constexpr (Cfg::kUpd)
            for (int q = 0; q < 4; ++q)
                for (int k = 0; k < kTpUpdSlots; ++k) tc_mbar_init(epi_full(q, k), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        if constexpr (Cfg::kUpd) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
        }
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc_smem(tmem_slot)),
                     "r"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    constexpr int kAStage0 = kTpAcc * kTcBN;  // TMEM column of stage 0's A

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            long long it = 0;
            TpUnit u;
            int g = 0;  // ring position
            while (tp_next(args, it, u)) {
                int mt, nt;
                tp_tile_mn(args, u.tile, mt, nt);
                const int m0 = mt * kTcBM, n0 = nt * kTcBN;
                for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
                    const int s = g % kTpStages;
                    const uint32_t ph = (uint32_t)((g / kTpStages) & 1);
                    tc_mbar_wait(empty(s), ph ^ 1);
                    tc_mbar_expect_tx(full(s), kTcTile + kTpBTile);
                    const int k0 = kb * kTcBK;
                    if constexpr (!A_MN)
                        tc_tma_2d(&tmA, full(s), tileA(s), k0, m0);
                    else
                        tc_tma_2d(&tmA, full(s), tileA(s), m0, k0);
                    if constexpr (!B_MN) {
                        tc_tma_2d(&tmB, full(s), tileB(s), k0, n0);
                    } else {
#pragma unroll
                        for (int q = 0; q < kTcBN / 32; ++q) tc_tma_2d(&tmB, full(s), tileB(s) + q * 4096, n0 + 32 * q, k0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((B_MN ? 1u : 0u) << 16) |
                               ((uint32_t)(kTcBN >> 3) << 17) | ((uint32_t)(kTcBM >> 4) << 24);
        long long it = 0;
        TpUnit u;
        int g = 0, n_unit = 0;
        while (tp_next(args, it, u)) {
            const int b = n_unit & 1;
            const uint32_t acc = tmem + (uint32_t)(b * kTcBN);
            tc_mbar_wait(acc_empty(b), (uint32_t)(((n_unit >> 1) & 1) ^ 1));  // the epilogue drained it
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
                const int s = g % kTpStages;
                const uint32_t ph = (uint32_t)((g / kTpStages) & 1);
                tc_mbar_wait(conv(s), ph);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                if (lane == 0) {
#pragma unroll
                    for (int ks = 0; ks < kTcBK / 8; ++ks) {
                        const uint32_t bo = B_MN ? ks * 1024u : ks * 32u;
                        const uint32_t blbo = B_MN ? 4096u : 16u, bsbo = B_MN ? 512u : 1024u, blay = B_MN ? 1u : 2u;
                        const uint64_t dB = tc_desc(tileB(s) + bo, blbo, bsbo, blay);
                        const uint64_t dBl = tc_desc(tileBlo(s) + bo, blbo, bsbo, blay);
                        const uint32_t tA = tmem + (uint32_t)(kAStage0 + 64 * s + 8 * ks);  // A; A_lo at +32
                        const uint32_t first = (kb == u.kb0 && ks == 0) ? 0u : 1u;
                        tc_mma_ts(acc, tA + 32u, dB, idesc, first);  // small terms first
                        tc_mma_ts(acc, tA, dBl, idesc, 1u);
                        tc_mma_ts(acc, tA, dB, idesc, 1u);
                    }
                    tc_commit(empty(s));
                }
                __syncwarp();
            }
            if (lane == 0) tc_commit(acc_full(b));
            __syncwarp();
            ++n_unit;
        }
    } else if (warp < 2 + kTpSplitWarps) {
        // ---------------- split pass ----------------
        const int ct = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int rowA = quarter * 32 + lane;
        const int khalf = (warp - 2) >> 2;
        long long it = 0;
        TpUnit u;
        int g = 0;
        while (tp_next(args, it, u)) {
            for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
                const int s = g % kTpStages;
                const uint32_t ph = (uint32_t)((g / kTpStages) & 1);
                tc_mbar_wait(full(s), ph);
                const uint8_t* a = smem + (size_t)s * kTpStage;
                const float4* bsrc = reinterpret_cast<const float4*>(smem + (size_t)s * kTpStage + kTcTile);
                float4* bl = reinterpret_cast<float4*>(smem + (size_t)s * kTpStage);  // B_lo over A
                uint32_t hi[16], lo[16];
                if constexpr (!A_MN) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int chunk = (4 * khalf + c) ^ (rowA & 7);
                        const float4 v = *reinterpret_cast<const float4*>(a + rowA * 128 + chunk * 16);
                        hi[4 * c + 0] = __float_as_uint(v.x);
                        hi[4 * c + 1] = __float_as_uint(v.y);
                        hi[4 * c + 2] = __float_as_uint(v.z);
                        hi[4 * c + 3] = __float_as_uint(v.w);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        hi[j] = __float_as_uint(*reinterpret_cast<const float*>(a + (16 * khalf + j) * 512 + rowA * 4));
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) lo[j] = __float_as_uint(tf32_lo(__uint_as_float(hi[j])));
                const uint32_t tA = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(kAStage0 + 64 * s + 16 * khalf);
                tc_st16(tA, hi);
                tc_st16(tA + 32u, lo);
                // every split warp has its A values in registers: B_lo may overwrite A
                asm volatile("bar.sync 2, %0;\n" ::"n"(32 * kTpSplitWarps) : "memory");
#pragma unroll
                for (int q = 0; q < kTpBTile / 16 / (32 * kTpSplitWarps); ++q) {
                    const int e = ct + 32 * kTpSplitWarps * q;
                    const float4 vb = bsrc[e];
                    bl[e] = make_float4(tf32_lo(vb.x), tf32_lo(vb.y), tf32_lo(vb.z), tf32_lo(vb.w));
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) tc_mbar_arrive(conv(s));
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const bool leader = warp == 2 + kTpSplitWarps && lane == 0;
        long long it = 0;
        TpUnit u;
        int n_unit = 0;
        if constexpr (Cfg::kUpd) {
            if (!args.sk) {
                // wgrad + update, whole tiles.  Each epilogue warp streams the W
                // and V sub-chunks of its own 32 rows (32 x 16 fp32, 64B swizzle,
                // 2 KB each): its lane 0 TMA-loads them kTpUpdSlots - 1 chunks
                // ahead -- across unit boundaries, i.e. during the next tile's
                // MMAs -- every lane updates its row in shared memory, G goes
                // straight to global, and lane 0 TMA-stores W and V back.  No
                // barrier across the epilogue warps: each runs its own pipeline.
                // (With one 128-row chunk per step shared by the 4 warps, a named
                // barrier per chunk serialised them: 57 us per C3 4096^2 wgrad.)
                constexpr int kChunks = kTcBN / kTpUpdCols;
                constexpr uint32_t kSub = 32 * kTpUpdCols * 4;  // one warp's W or V sub-chunk
                const uint32_t vbytes = args.mu == 0.0f ? 0u : kSub;
                uint8_t* const wbuf = epi_buf + (size_t)quarter * kTpUpdSlots * 2 * kSub;
                long long lit = 0;  // the loads' own cursor over units / chunks
                TpUnit lu;
                bool lmore = tp_next(args, lit, lu);
                int lchunk = 0, lissued = 0;
                auto issue_load = [&]() {  // lane 0: the next sub-chunk in unit order, if any
                    if (!lmore) return;
                    int mt, nt;
                    tp_tile_mn(args, lu.tile, mt, nt);
                    const int k = lissued % kTpUpdSlots;
                    const uint32_t wdst = tc_smem(wbuf + (size_t)(2 * k) * kSub);
                    const int r0 = mt * kTcBM + quarter * 32;
                    tc_mbar_expect_tx(epi_full(quarter, k), kSub + vbytes);
                    tc_tma_2d(&tmW, epi_full(quarter, k), wdst, nt * kTcBN + kTpUpdCols * lchunk, r0);
                    if (vbytes) tc_tma_2d(&tmV, epi_full(quarter, k), wdst + kSub, nt * kTcBN + kTpUpdCols * lchunk, r0);
                    ++lissued;
                    if (++lchunk == kChunks) {
                        lchunk = 0;
                        lmore = tp_next(args, lit, lu);
                    }
                };
                if (lane == 0)
                    for (int q = 0; q < kTpUpdSlots - 1; ++q) issue_load();
                int gc = 0;  // chunks consumed
                while (tp_next(args, it, u)) {
                    const int b = n_unit & 1;
                    tc_mbar_wait(acc_full(b), (uint32_t)((n_unit >> 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    int mt, nt;
                    tp_tile_mn(args, u.tile, mt, nt);
                    const int m = mt * kTcBM + row, n0 = nt * kTcBN;
                    const uint32_t tacc = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kTcBN);
#pragma unroll 1
                    for (int c = 0; c < kChunks; ++c, ++gc) {
                        float v[kTpUpdCols];
                        tp_ld16(tacc + (uint32_t)(kTpUpdCols * c), v);
                        if (c == kChunks - 1) {
                            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                            __syncwarp();
                            if (lane == 0) tc_mbar_arrive(acc_empty(b));
                        }
                        const int k = gc % kTpUpdSlots;
                        tc_mbar_wait(epi_full(quarter, k), (uint32_t)((gc / kTpUpdSlots) & 1));
                        uint8_t* wrow = wbuf + (size_t)(2 * k) * kSub + lane * (4 * kTpUpdCols);
                        uint8_t* vrow = wrow + kSub;
                        const bool full_cols = n0 + kTpUpdCols * c + kTpUpdCols <= args.N && (args.N & 3) == 0;
#pragma unroll
                        for (int q = 0; q < kTpUpdCols / 4; ++q) {
                            const int off = ((q ^ ((lane >> 1) & 3)) * 16);  // 64B swizzle: 16-byte unit q of row lane
                            float4 w = *reinterpret_cast<const float4*>(wrow + off);
                            float4 vv = args.mu == 0.0f ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                        : *reinterpret_cast<const float4*>(vrow + off);
                            float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                            float* xp = &x.x;
                            float* wp = &w.x;
                            float* vp = &vv.x;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float gg = smul(xp[i], args.inv_b);
                                xp[i] = gg;
                                const float step = smul(args.neg_eta, gg);
                                vp[i] = args.mu == 0.0f ? step : sadd(smul(args.mu, vp[i]), step);
                                wp[i] = sadd(wp[i], vp[i]);
                            }
                            *reinterpret_cast<float4*>(wrow + off) = w;
                            *reinterpret_cast<float4*>(vrow + off) = vv;
                            const int n = n0 + kTpUpdCols * c + 4 * q;
                            if (m < args.M) {
                                if (full_cols) {
                                    __stcs(reinterpret_cast<float4*>(args.C + (size_t)m * args.N + n), x);
                                } else {
                                    for (int i = 0; i < 4; ++i)
                                        if (n + i < args.N) args.C[(size_t)m * args.N + n + i] = xp[i];
                                }
                            }
                        }
                        // generic-proxy smem writes -> visible to the TMA store
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            const uint32_t wsrc = tc_smem(wbuf + (size_t)(2 * k) * kSub);
                            const int r0 = mt * kTcBM + quarter * 32;
                            tp_tma_store_2d(&tmW, wsrc, n0 + kTpUpdCols * c, r0);
                            tp_tma_store_2d(&tmV, wsrc + kSub, n0 + kTpUpdCols * c, r0);
                            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                            // the next load refills the previous chunk's slot, once
                            // that chunk's stores have read it (this chunk's may
                            // still be in flight)
                            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                            issue_load();
                        }
                        __syncwarp();
                    }
                    ++n_unit;
                }
                if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
            }
        }
        while (tp_next(args, it, u)) {
            const int b = n_unit & 1;
            tc_mbar_wait(acc_full(b), (uint32_t)((n_unit >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            int mt, nt;
            tp_tile_mn(args, u.tile, mt, nt);
            const int m = mt * kTcBM + row, n0 = nt * kTcBN;
            const uint32_t tacc = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kTcBN);
            if (u.npieces == 1) {
#pragma unroll 1
                for (int c = 0; c < kTcBN / 32; ++c) {
                    float v[32];
                    tp_ld32(tacc + (uint32_t)(32 * c), v);
                    if (c == kTcBN / 32 - 1) {
                        // the accumulator is in registers: hand it back to the MMA warp
                        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                        __syncwarp();
                        if (lane == 0) tc_mbar_arrive(acc_empty(b));
                    }
                    if (m < args.M) tp_epi_store<E>(args, m, n0 + 32 * c, v);
                }
            } else {
                // stream-K: the tile's pieces in K order; piece 0 (the one
                // holding K block 0) is its CTA's LAST unit, while the later
                // pieces open their CTAs' ranges, so piece 0 finishes the tile:
                // it waits until pieces 1.. have published their raw partials
                // (normally long done), then sums acc0 + acc1 + ... in piece
                // order (deterministic) and runs the fused epilogue.
                if (u.piece != 0) {
                    float* mine = args.part + ((size_t)u.tile * args.max_pieces + u.piece) * kTpTileElems +
                                  (size_t)row * kTcBN;
#pragma unroll 1
                    for (int c = 0; c < kTcBN / 32; ++c) {
                        float v[32];
                        tp_ld32(tacc + (uint32_t)(32 * c), v);
                        if (c == kTcBN / 32 - 1) {
                            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                            __syncwarp();
                            if (lane == 0) tc_mbar_arrive(acc_empty(b));
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            __stcg(reinterpret_cast<float4*>(mine + 32 * c + 4 * q),
                                   make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                    }
                    __threadfence();
                    tp_epi_bar();
                    if (leader) atomicAdd(args.counters + u.tile, 1);
                } else {
                    if (leader) {
                        const unsigned long long t0 = tp_globaltimer();
                        while (tp_ld_acquire(args.counters + u.tile) < u.npieces - 1) {
                            __nanosleep(100);
                            if (tp_globaltimer() - t0 > 5000000000ull) __trap();  // a lost piece: fail, never hang
                        }
                        args.counters[u.tile] = 0;  // ready for the next launch
                    }
                    tp_epi_bar();
                    const float* base = args.part + (size_t)u.tile * args.max_pieces * kTpTileElems + (size_t)row * kTcBN;
                    constexpr int kMaxP = 4;  // tp_plan keeps every tile within 4 pieces
#pragma unroll 1
                    for (int c = 0; c < kTcBN / 16; ++c) {
                        float v[16];
                        tp_ld16(tacc + (uint32_t)(16 * c), v);
                        if (c == kTcBN / 16 - 1) {
                            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                            __syncwarp();
                            if (lane == 0) tc_mbar_arrive(acc_empty(b));
                        }
                        float4 x[kMaxP - 1][4];
#pragma unroll
                        for (int p = 1; p < kMaxP; ++p)
                            if (p < u.npieces)
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    x[p - 1][q] = __ldcg(reinterpret_cast<const float4*>(
                                        base + (size_t)p * kTpTileElems + 16 * c + 4 * q));
#pragma unroll
                        for (int p = 1; p < kMaxP; ++p)
                            if (p < u.npieces)
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    v[4 * q] += x[p - 1][q].x;
                                    v[4 * q + 1] += x[p - 1][q].y;
                                    v[4 * q + 2] += x[p - 1][q].z;
                                    v[4 * q + 3] += x[p - 1][q].w;
                                }
                        if (m < args.M) tp_epi_store<E>(args, m, n0 + 16 * c, v);
                    }
                }
            }
            ++n_unit;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcTmemCols));
    }
}

}  // namespace lane_b200

// ---------------------------------------------------------------- host side
namespace lane_b200 {

struct TpPlan {
    int grid = 0;
    TpArgs a{};
    size_t part_floats = 0;  // stream-K workspace
    int tiles = 0;
};

// Decide data parallel vs stream-K for M x N x K on `sms` SMs.
inline TpPlan tp_plan(int M, int N, int K, int sms) {
    TpPlan p;
    TpArgs& a = p.a;
    a.M = M;
    a.N = N;
    a.K = K;
    a.tiles_m = (M + kTcBM - 1) / kTcBM;
    a.tiles_n = (N + kTcBN - 1) / kTcBN;
    a.kbs = (K + kTcBK - 1) / kTcBK;
    a.group = 8;
    p.tiles = a.tiles_m * a.tiles_n;
    const long long total = (long long)p.tiles * a.kbs;
    // whole tiles when the last wave is >= 85% full or there are many waves
    const int waves = (p.tiles + sms - 1) / sms;
    const double fill = (double)p.tiles / ((double)waves * sms);
    if (p.tiles >= 4 * sms || fill >= 0.85) {
        a.sk = 0;
        a.per = 0;
        a.max_pieces = 1;
        p.grid = std::min(p.tiles, sms);
    } else {
        a.sk = 1;
        a.per = (int)((total + sms - 1) / sms);
        // pieces shorter than 4 K blocks cost more in fix-up than they balance,
        // and the finishing piece sums at most 4 (per >= kbs / 3)
        a.per = std::max({a.per, std::min(a.kbs, 4), (a.kbs + 2) / 3});
        p.grid = (int)((total + a.per - 1) / a.per);
        a.max_pieces = (a.kbs + a.per - 1) / a.per + 1;
        p.part_floats = (size_t)p.tiles * a.max_pieces * kTpTileElems;
    }
    return p;
}

template <bool A_MN, bool B_MN, TpEpi E>
inline void tp_launch(cudaStream_t st, const CUtensorMap& ma, const CUtensorMap& mb, const TpPlan& p) {
    constexpr size_t smem = TpCfg<(int)E>::kSmem;
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    LANE_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        LANE_CUDA(cudaFuncSetAttribute(k_gemm_tcp<A_MN, B_MN, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured.fetch_or(bit, std::memory_order_release);
    }
    // UPDATE: W and V as [M rows x N cols] boxes of 32 rows x 16 columns
    // (64B swizzle) for each epilogue warp's TMA loads and stores
    const CUtensorMap mw = E == TpEpi::UPDATE ? tc_map(p.a.W, p.a.M, p.a.N, kTpUpdCols, 32, 3) : ma;
    const CUtensorMap mv = E == TpEpi::UPDATE ? tc_map(p.a.V, p.a.M, p.a.N, kTpUpdCols, 32, 3) : ma;
    k_gemm_tcp<A_MN, B_MN, E><<<p.grid, kTpThreads, smem, st>>>(ma, mb, mw, mv, p.a);
}

template <TpEpi E>
inline void tp_dispatch(cudaStream_t st, bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                        const TpPlan& p) {
    if (!a_mn && !b_mn) tp_launch<false, false, E>(st, ma, mb, p);
    else if (!a_mn && b_mn) tp_launch<false, true, E>(st, ma, mb, p);
    else if (a_mn && !b_mn) tp_launch<true, false, E>(st, ma, mb, p);
    else tp_launch<true, true, E>(st, ma, mb, p);
}

}  // namespace lane_b200
