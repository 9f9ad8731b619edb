// gemm_tc.cuh -- fp32-accurate GEMM on the 5th-generation tensor cores
// (tcgen05, kind::tf32) for the mini-batch path, "3xTF32":
//     A.B ~= A_lo.B + A.B_lo + A.B      (A_lo = A - tf32(A), exact in fp32)
// The tensor core reads fp32 operands and ignores their low 13 mantissa bits,
// so A itself is the "hi" part.  A is staged through tensor memory: the split
// warps read each TMA-loaded A tile once and write A and A_lo into TMEM
// (tcgen05.st); the MMAs take A from TMEM and B / B_lo from shared memory.
// Shared-memory traffic per 128x128x32 K block is then 128 KB (TMA 32, split
// reads 32 + B_lo writes 16, MMA operand reads 48) instead of 192 KB with both
// lo parts in shared memory -- the kernel was bound by the ~128 B/clk of SMEM
// bandwidth, not by the tensor pipe.  All three products accumulate into one
// fp32 TMEM accumulator.  Relative error per product ~2^-21 (the dropped A_lo.B_lo term
// and the tf32 truncation of the lo parts), within the path's 1e-5 tolerance
// (1xTF32 alone is ~5e-4 and is NOT used).
//
// Structure (one 128x128 output tile per CTA -- or one 256x256 tile per CTA
// pair, below -- 320 threads, 4-stage ring):
//   warp 0      TMA producer: A/B tiles (fp32) -> smem ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (A from
//               TMEM), commits smem/TMEM slots back to the producer and the
//               accumulator to the epilogue (tcgen05.commit -> mbarrier)
//   warps 2..9  split pass: rows of A -> TMEM (A, A_lo; the two warps of a
//               TMEM lane quarter take 16 K columns each) and B_lo -> smem;
//               then the epilogue (two warps per lane quarter, half the
//               tile's columns each): tcgen05.ld TMEM -> registers -> fused
//               epilogue -> global
// TMEM: columns [0, tile N) accumulator, then per stage 32 columns of A and 32
// of A_lo (lane = row of A, column = k).
// Operand majors: K-major tiles come from one TMA box {32 (K), 128 (MN)},
// 128B swizzle; a MN-major B from four boxes {32 (MN), 32 (K)} (32-byte-atom
// swizzle, the layout the MMA reads); a MN-major A -- read only by the split
// warps -- from one unswizzled box {128 (MN), 32 (K)}.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace lane_b200 {

constexpr int kTcBM = 128, kTcBN = 128, kTcBK = 32;
constexpr int kTcTile = kTcBM * kTcBK * 4;  // bytes of one 128x32 fp32 tile (A)
constexpr int kTcTmemCols = 512;            // accumulator (128) + stages x (A, A_lo) x 32
// Per-CTA ring.  PAIR = a CTA pair (cluster of 2, tcgen05 cta_group::2) on a
// 256 x 256 tile, issued as N = 256 MMAs: each CTA holds its 128 rows of A (in
// TMEM) and half (128 columns) of B; rank 0 issues the pair's MMAs.
template <bool PAIR>
struct TcCfg {
    static constexpr int kBN = PAIR ? 2 * kTcBN : kTcBN;   // tile N (pairs: 256 x 256 tiles)
    static constexpr int kBLocal = PAIR ? kBN / 2 : kBN;   // B columns this CTA holds
    static constexpr int kBTile = kBLocal * kTcBK * 4;
    static constexpr int kStage = kTcTile + 2 * kBTile;  // A, B, B_lo
    static constexpr int kStages = 4;                    // TMEM: kBN + 64 x stages <= 512
    static constexpr size_t kSmem = (size_t)kStages * kStage + 1024 /*align*/ + 512 /*barriers*/;
};
constexpr int kTcSplitWarps = 8;  // the split pass is the busiest role (3xTF32)
constexpr int kTcThreads = 64 + 32 * kTcSplitWarps;

enum class TcEpi : int { STORE = 0, BIAS = 1, BIAS_TANH = 2, TANH_GRAD = 3 };

struct TcArgs {
    int M, N, K;
    int kbs;            // split-K: K blocks per split (gridDim.z splits); 0 = no split
    float* part;        // split-K: raw partial tiles [split][M][N] (epilogue runs in the reduce)
    float* C;           // M x N row-major (ldc = N)
    float* C2;          // BIAS_TANH: tanh(C)
    const float* bias;  // BIAS*: per column
    const float* aux;   // TANH_GRAD: activations a (M x N)
    // 3xF16 kernel (gemm_h3.cuh): max |.| bits of every row of op(A) / column
    // of op(B), from which the power-of-two operand scales are derived
    const unsigned* amax = nullptr;
    const unsigned* bmax = nullptr;
    int diag = 0;  // experiments (LANE_B200_H3_DIAG): 1 skip the split math, 2 skip the MMAs, 4 / 8 skip the B / A loads
    // 3xF16 epilogue (optional): max |.| bits of every row / column of the
    // output operand the next GEMMs read (zeroed by the caller)
    unsigned* omax_row = nullptr;
    unsigned* omax_col = nullptr;
    // 3xF16 CTA pairs, tail-wave split: whole tiles [0, full_units), then the
    // two K halves of each remaining tile (raw partials in tail_part)
    int full_units = 0, tiles_m = 0, tiles_n = 0;
    float* tail_part = nullptr;
    // STORE (3xF16 wgrad of a one-rank step): C = sum * out_scale when non-zero
    // (the mean gradient; the update then neither rescales nor rewrites G)
    float out_scale = 0.0f;
};

// ---- PTX helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t tc_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tc_mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_tma_2d(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// UMMA shared-memory descriptor (sm100, version 1).  layout 2 = SWIZZLE_128B
// (K-major tiles); layout 1 = SWIZZLE_128B_BASE32B, the only smem layout the
// tensor core accepts for MN-major tf32 operands (32-byte swizzle atoms,
// 4-row groups; TMA side: CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t tc_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (Blackwell)
    d |= (uint64_t)layout << 61;
    return d;
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// A from tensor memory (K-major: lane = row, column = k), B from shared memory
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_mma_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
// arrive on the same-offset barrier of both CTAs of the pair once the MMAs
// issued so far have completed
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            bar),
        "h"((unsigned short)3)
        : "memory");
}
// release-arrive on the barrier at this CTA-local offset in cluster CTA `rank`
__device__ __forceinline__ void tc_mbar_arrive_remote(uint32_t local, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait_cluster(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAITC_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAITC_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// 32 lanes x 16 consecutive 32-bit TMEM columns from registers
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}

// low part of a tf32 split: x - (x with the 13 low mantissa bits cleared)
__device__ __forceinline__ float tf32_lo(float x) {
    return __fsub_rn(x, __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}

template <TcEpi E>
__device__ __forceinline__ float4 tc_epi4(const TcArgs& a, int m, int n, float4 v, float4* second) {
    if constexpr (E == TcEpi::BIAS || E == TcEpi::BIAS_TANH) {
        const float4 b = *reinterpret_cast<const float4*>(a.bias + n);
        v.x = sadd(v.x, b.x);
        v.y = sadd(v.y, b.y);
        v.z = sadd(v.z, b.z);
        v.w = sadd(v.w, b.w);
        if constexpr (E == TcEpi::BIAS_TANH) {
            second->x = tanhf(v.x);  // FAST numerics: libdevice tanhf (<= 2 ulp)
            second->y = tanhf(v.y);
            second->z = tanhf(v.z);
            second->w = tanhf(v.w);
        }
    } else if constexpr (E == TcEpi::TANH_GRAD) {
        const float4 t = *reinterpret_cast<const float4*>(a.aux + (size_t)m * a.N + n);
        v.x = tanh_grad(t.x, v.x);
        v.y = tanh_grad(t.y, v.y);
        v.z = tanh_grad(t.z, v.z);
        v.w = tanh_grad(t.w, v.w);
    } else if constexpr (E == TcEpi::STORE) {
        if (a.out_scale != 0.0f) {
            v.x = smul(v.x, a.out_scale);
            v.y = smul(v.y, a.out_scale);
            v.z = smul(v.z, a.out_scale);
            v.w = smul(v.w, a.out_scale);
        }
    }
    return v;
}

template <bool A_MN, bool B_MN, TcEpi E, bool PAIR>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs args) {
    using Cfg = TcCfg<PAIR>;
    constexpr int kTcStages = Cfg::kStages, kTcStage = Cfg::kStage, kBTile = Cfg::kBTile;
    extern __shared__ uint8_t tc_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kTcStages * kTcStage);
    // bars: full[S], conv[S], empty[S], tmem_full[1]; then the TMEM address
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // PAIR: cluster (2,1,1) along x = M; rank 0 issues the pair's MMAs
    const uint32_t rank = PAIR ? (blockIdx.x & 1u) : 0u;
    const int m0 = PAIR ? (int)(blockIdx.x >> 1) * 2 * kTcBM + (int)rank * kTcBM : (int)blockIdx.y * kTcBM;
    const int n0 = PAIR ? (int)blockIdx.y * Cfg::kBN : (int)blockIdx.x * kTcBN;
    // split-K: this CTA accumulates K blocks [kb0, kb1)
    const int nkb_all = (args.K + kTcBK - 1) / kTcBK;
    const int kb0 = gridDim.z > 1 ? blockIdx.z * args.kbs : 0;
    const int kb1 = gridDim.z > 1 ? min(nkb_all, kb0 + args.kbs) : nkb_all;
    const int nkb = kb1 - kb0;
    const bool split = gridDim.z > 1;
    const uint32_t sbase = tc_smem(smem);
    auto full = [&](int s) { return tc_smem(bars + s); };
    auto conv = [&](int s) { return tc_smem(bars + kTcStages + s); };
    auto empty = [&](int s) { return tc_smem(bars + 2 * kTcStages + s); };
    const uint32_t tmem_full = tc_smem(bars + 3 * kTcStages);
    auto tileA = [&](int s) { return sbase + (uint32_t)(s * kTcStage); };
    auto tileB = [&](int s) { return sbase + (uint32_t)(s * kTcStage + kTcTile); };
    auto tileBlo = [&](int s) { return sbase + (uint32_t)(s * kTcStage + kTcTile + kBTile); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            tc_mbar_init(full(s), 1);
            // PAIR: rank 1's "split done" reaches rank 0's conv(s) as the
            // complete_tx of a 16-byte DSMEM bulk copy (one of rank 0's split
            // warps arms the matching expect_tx) -- no cluster-scope fence
            tc_mbar_init(conv(s), kTcSplitWarps);
            tc_mbar_init(empty(s), 1);
        }
        tc_mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             tc_smem(tmem_slot)),
                         "r"(kTcTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             tc_smem(tmem_slot)),
                         "r"(kTcTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (PAIR)
        tc_cluster_sync();  // both CTAs' barriers initialised before any remote arrive / multicast commit
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kTcStages;
                const uint32_t ph = (uint32_t)((kb / kTcStages) & 1);
                tc_mbar_wait(empty(s), ph ^ 1);
                tc_mbar_expect_tx(full(s), kTcTile + kBTile);
                const int k0 = (kb0 + kb) * kTcBK;
                if constexpr (!A_MN)
                    tc_tma_2d(&tmA, full(s), tileA(s), k0, m0);
                else
                    tc_tma_2d(&tmA, full(s), tileA(s), m0, k0);  // unswizzled [k][128 m]
                const int nb = n0 + (int)rank * Cfg::kBLocal;  // this CTA's B columns
                if constexpr (!B_MN) {
                    tc_tma_2d(&tmB, full(s), tileB(s), k0, nb);
                } else {
#pragma unroll
                    for (int g = 0; g < Cfg::kBLocal / 32; ++g)
                        tc_tma_2d(&tmB, full(s), tileB(s) + g * 4096, nb + 32 * g, k0);
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer ----------------
        // instruction descriptor: D f32, A/B tf32, A K-major (TMEM), B major, N>>3, M>>4
        constexpr uint32_t kM = PAIR ? 2 * kTcBM : kTcBM;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((B_MN ? 1u : 0u) << 16) |
                               ((uint32_t)(Cfg::kBN >> 3) << 17) | ((kM >> 4) << 24);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (uint32_t)((kb / kTcStages) & 1);
            tc_mbar_wait(conv(s), ph);  // PAIR: both CTAs' split passes (rank 1's forwarded)
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (lane == 0) {
#pragma unroll
                for (int ks = 0; ks < kTcBK / 8; ++ks) {
                    // B: K-major +32 B inside the 128 B swizzle row (SBO = 8 rows x
                    // 128 B); MN-major SW128_BASE32B +8 K-rows (LBO = 32-wide MN
                    // group, one TMA box; SBO = 4 K-rows x 128 B)
                    const uint32_t bo = B_MN ? ks * 1024u : ks * 32u;
                    const uint32_t blbo = B_MN ? 4096u : 16u, bsbo = B_MN ? 512u : 1024u, blay = B_MN ? 1u : 2u;
                    const uint64_t dB = tc_desc(tileB(s) + bo, blbo, bsbo, blay);
                    const uint64_t dBl = tc_desc(tileBlo(s) + bo, blbo, bsbo, blay);
                    const uint32_t tA = tmem + (uint32_t)(Cfg::kBN + 64 * s + 8 * ks);  // A; A_lo at +32
                    const uint32_t first = (kb == 0 && ks == 0) ? 0u : 1u;
                    if constexpr (PAIR) {
                        tc_mma_ts_pair(tmem, tA + 32u, dB, idesc, first);  // small terms first
                        tc_mma_ts_pair(tmem, tA, dBl, idesc, 1u);
                        tc_mma_ts_pair(tmem, tA, dB, idesc, 1u);
                    } else {
                        tc_mma_ts(tmem, tA + 32u, dB, idesc, first);  // small terms first
                        tc_mma_ts(tmem, tA, dBl, idesc, 1u);
                        tc_mma_ts(tmem, tA, dB, idesc, 1u);
                    }
                }
                // slot free (in both CTAs) once these MMAs have read it
                if constexpr (PAIR)
                    tc_commit_pair(empty(s));
                else
                    tc_commit(empty(s));
            }
            __syncwarp();
        }
        if (lane == 0) {
            if constexpr (PAIR)
                tc_commit_pair(tmem_full);
            else
                tc_commit(tmem_full);
        }
        __syncwarp();
    } else if (warp == 1) {
        // the pair's second CTA: its MMAs are issued by rank 0.  This warp
        // forwards "stage s split done" to rank 0 as an async-proxy DSMEM bulk
        // copy that completes rank 0's conv(s) transaction count.
        if (lane == 0) {
            const uint32_t src = tc_smem(reinterpret_cast<uint8_t*>(bars) + 464);
            uint32_t dst, rbar0;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(dst) : "r"(src - 16), "r"(0));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbar0) : "r"(conv(0)), "r"(0));
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kTcStages;
                const uint32_t ph = (uint32_t)((kb / kTcStages) & 1);
                tc_mbar_wait(conv(s), ph);
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];\n" ::"r"(
                        dst),
                    "r"(src), "r"(rbar0 + 8u * (uint32_t)s)
                    : "memory");
            }
        }
        __syncwarp();
    } else {
        // ---------------- split pass, then epilogue (warps 2..9) ----------------
        const int ct = threadIdx.x - 64;  // 0..32*kTcSplitWarps-1
        const int quarter_s = warp & 3;   // TMEM lanes this warp may access
        const int rowA = quarter_s * 32 + lane;
        const int khalf = (warp - 2) >> 2;  // K columns [16 khalf, 16 khalf + 16) of the block
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (uint32_t)((kb / kTcStages) & 1);
            tc_mbar_wait(full(s), ph);
            const uint8_t* a = smem + (size_t)s * kTcStage;
            const float4* b = reinterpret_cast<const float4*>(smem + (size_t)s * kTcStage + kTcTile);
            float4* bl = reinterpret_cast<float4*>(smem + (size_t)s * kTcStage + kTcTile + kBTile);
            // A row rowA, K columns [16 khalf, +16) -> TMEM (A and A_lo)
            uint32_t hi[16], lo[16];
            if constexpr (!A_MN) {
                // SW128: 16-byte chunk c of row r sits at chunk c ^ (r & 7)
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
                // unswizzled [k][128 m]
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    hi[j] = __float_as_uint(*reinterpret_cast<const float*>(a + (16 * khalf + j) * 512 + rowA * 4));
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) lo[j] = __float_as_uint(tf32_lo(__uint_as_float(hi[j])));
            const uint32_t tA =
                tmem + ((uint32_t)(quarter_s * 32) << 16) + (uint32_t)(Cfg::kBN + 64 * s + 16 * khalf);
            tc_st16(tA, hi);
            tc_st16(tA + 32u, lo);
            // B_lo -> smem (same swizzled layout as B)
#pragma unroll
            for (int u = 0; u < kBTile / 16 / (32 * kTcSplitWarps); ++u) {
                const int q = ct + 32 * kTcSplitWarps * u;
                const float4 vb = b[q];
                bl[q] = make_float4(tf32_lo(vb.x), tf32_lo(vb.y), tf32_lo(vb.z), tf32_lo(vb.w));
            }
            // TMEM stores complete + generic-proxy smem writes visible to the
            // tensor core (async proxy) before the MMA issuer is released
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (PAIR && rank == 0 && warp == 2)
                    tc_mbar_expect_tx(conv(s), 16);  // rank 1's forward (16-byte bulk copy)
                else
                    tc_mbar_arrive(conv(s));
            }
        }
        tc_mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int quarter = warp & 3;  // TMEM lanes this warp may access
        const int row = quarter * 32 + lane;
        const int cbeg = ((warp - 2) >> 2) * (Cfg::kBN / 2);  // this warp's half of the columns
        const int m = m0 + row;
#pragma unroll 1
        for (int c0 = cbeg; c0 < cbeg + Cfg::kBN / 2; c0 += 32) {
            uint32_t r[32];
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (m < args.M && split) {
                // raw partial; bias/activation are applied by k_tc_splitk_reduce
                float* P = args.part + (size_t)blockIdx.z * args.M * args.N + (size_t)m * args.N;
                const int nb = n0 + c0;
                if (nb + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(P + nb)[q] =
                            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                } else {
                    for (int q = 0; q < 32; ++q)
                        if (nb + q < args.N) P[nb + q] = __uint_as_float(r[q]);
                }
            } else if (m < args.M) {
                const int nb = n0 + c0;
                if (nb + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                               __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                        float4 t;
                        v = tc_epi4<E>(args, m, nb + 4 * q, v, &t);
                        *reinterpret_cast<float4*>(args.C + (size_t)m * args.N + nb + 4 * q) = v;
                        if constexpr (E == TcEpi::BIAS_TANH)
                            *reinterpret_cast<float4*>(args.C2 + (size_t)m * args.N + nb + 4 * q) = t;
                    }
                } else {
                    for (int q = 0; q < 32; ++q) {
                        const int n = nb + q;
                        if (n >= args.N) break;
                        float v = __uint_as_float(r[q]);
                        const size_t idx = (size_t)m * args.N + n;
                        if constexpr (E == TcEpi::BIAS || E == TcEpi::BIAS_TANH) v = sadd(v, args.bias[n]);
                        if constexpr (E == TcEpi::TANH_GRAD) v = tanh_grad(args.aux[idx], v);
                        args.C[idx] = v;
                        if constexpr (E == TcEpi::BIAS_TANH) args.C2[idx] = tanhf(v);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (PAIR)
        tc_cluster_sync();
    else
        __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcTmemCols));
    }
}

// C = epilogue(sum_z part[z]) in a fixed split order (deterministic); N % 4 == 0
template <TcEpi E>
__global__ void __launch_bounds__(256) k_tc_splitk_reduce(TcArgs a, int S) {
    const size_t n4 = (size_t)a.M * a.N / 4;
    const float4* P = reinterpret_cast<const float4*>(a.part);
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (size_t)gridDim.x * blockDim.x) {
        float4 v = P[e];
        for (int z = 1; z < S; ++z) {
            const float4 p = P[(size_t)z * n4 + e];
            v.x += p.x;
            v.y += p.y;
            v.z += p.z;
            v.w += p.w;
        }
        // 32-bit index math (M * N < 2^32 for every split-K shape): no 64-bit
        // division per element
        const unsigned q = (unsigned)(4 * e), uN = (unsigned)a.N;
        const int m = (int)(q / uN), n = (int)(q - (q / uN) * uN);
        float4 t;
        v = tc_epi4<E>(a, m, n, v, &t);
        reinterpret_cast<float4*>(a.C)[e] = v;
        if constexpr (E == TcEpi::BIAS_TANH) reinterpret_cast<float4*>(a.C2)[e] = t;
    }
}

}  // namespace lane_b200

// ---------------------------------------------------------------- host side
#include <cuda_runtime.h>

#include <atomic>

namespace lane_b200 {

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled tc_encoder() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        LANE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(LANE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

// 2-D fp32 row-major tensor [rows x cols] (ld = cols), box {box_inner, box_rows};
// swizzle: 0 = 128B (K-major MMA operand), 1 = 128B with 32-byte atoms (the
// MN-major tf32 MMA operand), 2 = none (read by the split warps only), 3 = 64B
// (the update epilogue's 16-column W / V chunks)
inline CUtensorMap tc_map(const float* base, int rows, int cols, int box_inner, int box_rows, int swizzle) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = tc_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    swizzle == 1   ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                    : swizzle == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                    : swizzle == 3 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(LANE_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

// The tensor-core path needs 16-byte row strides for every TMA operand.
inline bool tc_eligible(int M, int N, int K) {
    return (M % 4 == 0) && (N % 4 == 0) && (K % 4 == 0) && N >= 64 && M >= 64 && K >= 32;
}

template <bool A_MN, bool B_MN, TcEpi E, bool PAIR>
inline void tc_launch(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const TcArgs& args) {
    constexpr size_t smem = TcCfg<PAIR>::kSmem;
    // the attribute is per-device function state: set it once per device
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    LANE_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        LANE_CUDA(cudaFuncSetAttribute(k_gemm_tc<A_MN, B_MN, E, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured.fetch_or(bit, std::memory_order_release);
    }
    const int S = args.kbs > 0 ? (args.K / kTcBK + args.kbs - 1) / args.kbs : 1;
    if constexpr (PAIR) {
        // clusters of 2 along x (M): CTA 2p and 2p+1 share the 256 x 128 tile p
        cudaLaunchConfig_t cfg = {};
        constexpr int kBN = TcCfg<true>::kBN;
        cfg.gridDim = dim3(2 * ((args.M + 2 * kTcBM - 1) / (2 * kTcBM)), (args.N + kBN - 1) / kBN, S);
        cfg.blockDim = dim3(kTcThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LANE_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_tc<A_MN, B_MN, E, PAIR>, a, b, args));
    } else {
        const dim3 grid((args.N + kTcBN - 1) / kTcBN, (args.M + kTcBM - 1) / kTcBM, S);
        k_gemm_tc<A_MN, B_MN, E, PAIR><<<grid, kTcThreads, smem, st>>>(a, b, args);
    }
    if (S > 1) {
        const size_t n4 = (size_t)args.M * args.N / 4;
        k_tc_splitk_reduce<E><<<(unsigned)std::min<size_t>(1184, (n4 + 255) / 256), 256, 0, st>>>(args, S);
    }
}

template <TcEpi E, bool PAIR>
inline void tc_dispatch(cudaStream_t st, bool a_mn, bool b_mn, const CUtensorMap& a, const CUtensorMap& b,
                        const TcArgs& args) {
    if (!a_mn && !b_mn) tc_launch<false, false, E, PAIR>(st, a, b, args);
    else if (!a_mn && b_mn) tc_launch<false, true, E, PAIR>(st, a, b, args);
    else if (a_mn && !b_mn) tc_launch<true, false, E, PAIR>(st, a, b, args);
    else tc_launch<true, true, E, PAIR>(st, a, b, args);
}

}  // namespace lane_b200
