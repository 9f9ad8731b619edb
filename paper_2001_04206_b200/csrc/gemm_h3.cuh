// gemm_h3.cuh -- fp32-accurate GEMM on the tcgen05 tensor cores at the FP16
// rate, "3xF16": every operand element x is scaled by a power of two and split
// into two halves,
//     s x = hi + lo,   hi = f16(s x),   lo = f16(s x - hi)
// and the product is accumulated in fp32 as A_lo.B_hi + A_hi.B_lo + A_hi.B_hi
// (the dropped A_lo.B_lo term is ~2^-22 relative).  kind::f16 MMAs run at twice
// the kind::tf32 rate and read half the operand bytes, so the three products
// cost what 1.5 tf32 MMAs cost -- against 3 for the 3xTF32 kernel
// (gemm_tc.cuh), which was bound by the tensor pipe.
//
// Scales.  fp16 has 5 exponent bits, so each row m of op(A) is scaled by
// sa[m] = 2^(14 - e) with e the exponent of max_k |A[m][k]| (so the row's
// largest element lands in [2^14, 2^15) and nothing overflows), and each column
// n of op(B) by sb[n] likewise.  The scales are constant along K, so the MMA
// accumulates sa[m] sb[n] (A.B)[m][n] exactly as it would A.B, and the
// epilogue multiplies by the two inverse powers of two (exact).  An element
// 2^17 below its row's (column's) maximum still keeps a normal lo part; the
// precision degrades only gradually below that (subnormal lo), far beyond what
// the condition-aware 1e-5 bound can see.  The per-row / per-column maxima come
// from a one-pass pre-kernel (k_absmax_rows / k_absmax_cols, below).
//
// Structure: gemm_tc.cuh's (one 128 x 128 tile per CTA, or 256 x 256 per CTA
// pair with cta_group::2 and N = 256 MMAs; TMA producer, MMA issuer, 16 split
// warps that then run the epilogue).  Per 32-wide K block the split warps read
// the TMA-loaded fp32 A and B tiles (a 4-slot landing ring, released as soon
// as it is read) and write
//   A_hi, A_lo -> TMEM (lane = row, 32-bit column = a pair of K elements),
//   B_hi, B_lo -> shared memory, K-major, no swizzle (8 x 16-byte core
//                 matrices: LBO = 128 B along K, SBO = 512 B along N).
// into a 6-slot f16 ring.  Per K block the MMA issuer issues 2 K-steps
// (K = 16) x 3 MMAs.  Shared memory: landing slots 32 KB (A, B fp32), f16
// slots 16 KB (B_hi, B_lo).
// TMEM: accumulator [0, tile N), then per stage 16 columns of A_hi and 16 of A_lo.
#pragma once

#include <cuda_fp16.h>

#include "gemm_tc.cuh"

namespace lane_b200 {

// 16 split warps (4 per SM sub-partition) in two groups of 8 that take
// alternate K blocks (see the split loop)
constexpr int kH3SplitWarps = 16;
#ifndef LANE_H3_RASTER
#define LANE_H3_RASTER 8
#endif
constexpr int kH3Group = LANE_H3_RASTER;  // raster group (pair tile rows)
#ifndef LANE_H3_GROUPS
#define LANE_H3_GROUPS 4
#endif
constexpr int kH3Groups = LANE_H3_GROUPS;  // split-warp groups, each on its own K blocks
constexpr int kH3Threads = 64 + 32 * kH3SplitWarps;

template <bool PAIR>
struct H3Cfg {
    static constexpr int kBN = PAIR ? 2 * kTcBN : kTcBN;
    static constexpr int kBLocal = PAIR ? kBN / 2 : kBN;  // 128 B columns per CTA
    static constexpr int kA32 = kTcBM * kTcBK * 4;        // fp32 A tile
    static constexpr int kB32 = kBLocal * kTcBK * 4;      // fp32 B tile
    static constexpr int kB16 = kBLocal * kTcBK * 2;      // one f16 B part
    // two rings: fp32 landing slots (TMA -> split warps, freed as soon as they
    // are read) and f16 slots (split warps -> MMA, freed by the MMA commit), so
    // the TMA runs up to kLand + kStages K blocks ahead of the tensor core
    // (4 + 6 measured ~2% faster at 4096^3 than 5 + 4 or 3 + 8)
    static constexpr int kLand = 4, kStages = 6;
    static constexpr int kLandBytes = kA32 + kB32, kF16Bytes = 2 * kB16;
    static constexpr size_t kSmem = (size_t)kLand * kLandBytes + (size_t)kStages * kF16Bytes + 1024 + 512;
};

// power-of-two operand scale from the max |x| bits of a row / column: the
// maximum lands in [2^14, 2^15) (zero rows: exponent clamped, any scale works)
__device__ __forceinline__ int h3_exp(unsigned maxbits) {
    int e = (int)((maxbits >> 23) & 0xFFu) - 127;
    return e < -100 ? -100 : e;
}
__device__ __forceinline__ float h3_pow2(int p) { return __int_as_float((127 + p) << 23); }

// s*x split into f16 hi + lo, packed pairwise (k even in the low half).  hi is
// s*x truncated to 11 significant bits in fp32 (exactly an f16 for the scaled
// range [2^-14, 2^15)), so lo = s*x - hi is exact and no f16 -> f32
// conversion is needed; one packed cvt per pair for each part.
__device__ __forceinline__ uint32_t h3_pack(float lo_k, float hi_k) {
    uint32_t d;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(d) : "f"(hi_k), "f"(lo_k));  // hi_k -> upper half
    return d;
}
__device__ __forceinline__ void h3_split2(float x0, float x1, float s, uint32_t& hi, uint32_t& lo) {
    const float a0 = x0 * s, a1 = x1 * s;  // exact: power-of-two scale
    const float h0 = __uint_as_float(__float_as_uint(a0) & 0xFFFFE000u);
    const float h1 = __uint_as_float(__float_as_uint(a1) & 0xFFFFE000u);
    hi = h3_pack(h0, h1);
    lo = h3_pack(__fsub_rn(a0, h0), __fsub_rn(a1, h1));
}

__device__ __forceinline__ void h3_mma(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void h3_mma_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
// 32 lanes x 8 consecutive 32-bit TMEM columns from registers
__device__ __forceinline__ void h3_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void h3_sts4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// TMA store of one 2-D box from shared memory (bulk group)
__device__ __forceinline__ void h3_tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}

// 16 consecutive K values of one row (K-major SW128 fp32 tile, 128-byte rows)
// or of one column (MN-major unswizzled [32 k][128] fp32 tile); t is a
// shared-window address (explicit ld.shared: no generic-address loads)
template <bool MN>
__device__ __forceinline__ void h3_load16(uint32_t t, int r, int khalf, float (&v)[16]) {
    if constexpr (!MN) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int chunk = (4 * khalf + c) ^ (r & 7);
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                         : "=f"(v[4 * c]), "=f"(v[4 * c + 1]), "=f"(v[4 * c + 2]), "=f"(v[4 * c + 3])
                         : "r"(t + (uint32_t)(r * 128 + chunk * 16)));
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v[j]) : "r"(t + (uint32_t)((16 * khalf + j) * 512 + r * 4)));
    }
}

// pair tile t -> (tile row, tile column): grouped raster, kH3Group tile rows
// at a time, so a wave of 74 pairs covers an ~8 x 9 block of tiles and
// re-reads fewer A panels than row-major waves that sweep every tile row
__device__ __forceinline__ void h3_tile_mn(int t, int tiles_m, int tiles_n, int& mt, int& nt) {
    const int per_group = kH3Group * tiles_n;
    const int g = t / per_group, first = g * kH3Group;
    const int gm = min(tiles_m - first, kH3Group);
    const int rr = t - g * per_group;
    mt = first + rr % gm;
    nt = rr / gm;
}

template <bool A_MN, bool B_MN, TcEpi E, bool PAIR>
__global__ void __launch_bounds__(kH3Threads, 1)
    k_gemm_h3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2, TcArgs args) {
    using Cfg = H3Cfg<PAIR>;
    constexpr int kS = Cfg::kStages, kL = Cfg::kLand;
    extern __shared__ uint8_t h3_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(h3_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem + (size_t)kL * Cfg::kLandBytes + (size_t)kS * Cfg::kF16Bytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? (blockIdx.x & 1u) : 0u;
    // grouped raster: consecutive pair tiles (launch order) walk kH3Group
    // tile rows before the next tile column, so a wave of 74 pairs covers an
    // ~8 x 9 block of tiles and re-reads far fewer A panels from DRAM than
    // row-major waves that each sweep every tile row
    int mt, nt;
    // tail-wave split (pairs, args.full_units > 0): a 1-D grid of units; the
    // first full_units are whole tiles, the rest are the two K halves of the
    // last partial wave's tiles, written raw to args.tail_part and finished
    // by k_h3_tail_reduce -- the last wave then takes half a wave's time
    int tail = -1;  // tail unit: 2 * (tile - full_units) + half
    int tile;
    if constexpr (PAIR) {
        const int u = (int)(blockIdx.x >> 1) + (int)blockIdx.y * (int)(gridDim.x >> 1);
        if (args.full_units > 0 && u >= args.full_units) {
            tail = u - args.full_units;
            tile = args.full_units + (tail >> 1);
        } else {
            tile = u;
        }
        const int tiles_m = args.full_units > 0 ? args.tiles_m : (int)(gridDim.x >> 1);
        const int tiles_n = args.full_units > 0 ? args.tiles_n : (int)gridDim.y;
        h3_tile_mn(tile, tiles_m, tiles_n, mt, nt);
    } else {
        mt = (int)blockIdx.y;
        nt = (int)blockIdx.x;
        tile = 0;
    }
    const int m0 = PAIR ? mt * 2 * kTcBM + (int)rank * kTcBM : mt * kTcBM;
    const int n0 = nt * Cfg::kBN;
    const int nbl = n0 + (int)rank * Cfg::kBLocal;  // this CTA's B columns
    const int nkb_all = (args.K + kTcBK - 1) / kTcBK;
    int kb0 = gridDim.z > 1 ? blockIdx.z * args.kbs : 0;
    int kb1 = gridDim.z > 1 ? min(nkb_all, kb0 + args.kbs) : nkb_all;
    if (tail >= 0) {
        kb0 = (tail & 1) ? nkb_all / 2 : 0;
        kb1 = (tail & 1) ? nkb_all : nkb_all / 2;
    }
    const int nkb = kb1 - kb0;
    const bool split = gridDim.z > 1;
    const uint32_t sbase = tc_smem(smem);
    // barriers: full[kL] (TMA -> split), lempty[kL] (split -> TMA), conv[kS]
    // (split -> MMA), fempty[kS] (MMA -> split), tmem_full
    auto full = [&](int l) { return tc_smem(bars + l); };
    auto lempty = [&](int l) { return tc_smem(bars + kL + l); };
    auto conv = [&](int s) { return tc_smem(bars + 2 * kL + s); };
    auto fempty = [&](int s) { return tc_smem(bars + 2 * kL + kS + s); };
    const uint32_t tmem_full = tc_smem(bars + 2 * kL + 2 * kS);
    auto landA = [&](int l) { return sbase + (uint32_t)(l * Cfg::kLandBytes); };
    auto landB = [&](int l) { return sbase + (uint32_t)(l * Cfg::kLandBytes + Cfg::kA32); };
    const uint32_t f16base = sbase + (uint32_t)(kL * Cfg::kLandBytes);
    auto tileBh = [&](int s) { return f16base + (uint32_t)(s * Cfg::kF16Bytes); };
    auto tileBl = [&](int s) { return f16base + (uint32_t)(s * Cfg::kF16Bytes + Cfg::kB16); };

    if (threadIdx.x == 0) {
        for (int l = 0; l < kL; ++l) {
            tc_mbar_init(full(l), 1);
            tc_mbar_init(lempty(l), kH3SplitWarps / kH3Groups);  // one group per K block
        }
        for (int s = 0; s < kS; ++s) {
            tc_mbar_init(conv(s), kH3SplitWarps / kH3Groups);  // one group per K block
            tc_mbar_init(fempty(s), 1);
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
        tc_cluster_sync();
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer: fp32 A and B tiles ----------------
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int l = kb % kL;
                const uint32_t ph = (uint32_t)((kb / kL) & 1);
                tc_mbar_wait(lempty(l), ph ^ 1);
                const bool ldA = !(args.diag & 8), ldB = !(args.diag & 4);  // experiments only
                tc_mbar_expect_tx(full(l), (ldA ? Cfg::kA32 : 0) + (ldB ? Cfg::kB32 : 0));
                const int k0 = (kb0 + kb) * kTcBK;
                if (ldA) {
                    if constexpr (!A_MN)
                        tc_tma_2d(&tmA, full(l), landA(l), k0, m0);
                    else
                        tc_tma_2d(&tmA, full(l), landA(l), m0, k0);
                }
                if (ldB) {
                    if constexpr (!B_MN)
                        tc_tma_2d(&tmB, full(l), landB(l), k0, nbl);
                    else
                        tc_tma_2d(&tmB, full(l), landB(l), nbl, k0);
                }
            }
            if constexpr (E == TcEpi::TANH_GRAD && PAIR) {
                // the dgrad epilogue's activations (tmC2 maps aux): this CTA's
                // 128 rows x 256 columns into the landing ring as its slots free
                // up, during the last K blocks' MMAs.  Slot j = the 64 columns
                // [64 j, 64 j + 64) of epilogue warp group j: two 32-column
                // halves x 4 row quarters, one 32 x 32 box (4 KB, 128B swizzle) each.
                if (!split && tail < 0) {
                    for (int j = 0; j < kL; ++j) {
                        const int kb = nkb + j, l = kb % kL;
                        tc_mbar_wait(lempty(l), (uint32_t)(((kb / kL) & 1) ^ 1));
                        tc_mbar_expect_tx(full(l), (uint32_t)Cfg::kLandBytes);
                        for (int cc = 0; cc < 2; ++cc)
                            for (int q = 0; q < 4; ++q)
                                tc_tma_2d(&tmC2, full(l), landA(l) + (uint32_t)(cc * 16384 + q * 4096),
                                          n0 + 32 * (2 * j + cc), m0 + 32 * q);
                    }
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer ----------------
        // instruction descriptor: D f32, A/B f16, both K-major, N>>3, M>>4
        constexpr uint32_t kM = PAIR ? 2 * kTcBM : kTcBM;
        constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(Cfg::kBN >> 3) << 17) | ((kM >> 4) << 24);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kS;
            const uint32_t ph = (uint32_t)((kb / kS) & 1);
            tc_mbar_wait(conv(s), ph);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (lane == 0 && !(args.diag & 2)) {
#pragma unroll
                for (int ks = 0; ks < kTcBK / 16; ++ks) {
                    // no swizzle, K-major: core matrices 8 rows x 16 B; the K = 16
                    // step covers two of them (LBO = 128 B), 8-row groups at 512 B
                    const uint64_t dBh = tc_desc(tileBh(s) + 256u * ks, 128u, 512u, 0u);
                    const uint64_t dBl = tc_desc(tileBl(s) + 256u * ks, 128u, 512u, 0u);
                    const uint32_t tA = tmem + (uint32_t)(Cfg::kBN + 32 * s + 8 * ks);  // A_hi; A_lo at +16
                    const uint32_t first = (kb == 0 && ks == 0) ? 0u : 1u;
                    if constexpr (PAIR) {
                        h3_mma_pair(tmem, tA + 16u, dBh, idesc, first);  // small terms first
                        h3_mma_pair(tmem, tA, dBl, idesc, 1u);
                        h3_mma_pair(tmem, tA, dBh, idesc, 1u);
                    } else {
                        h3_mma(tmem, tA + 16u, dBh, idesc, first);
                        h3_mma(tmem, tA, dBl, idesc, 1u);
                        h3_mma(tmem, tA, dBh, idesc, 1u);
                    }
                }
            }
            if (lane == 0) {
                if constexpr (PAIR)
                    tc_commit_pair(fempty(s));
                else
                    tc_commit(fempty(s));
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
        // the pair's second CTA: forward "stage s split done" to rank 0 (see gemm_tc.cuh)
        if (lane == 0) {
            const uint32_t src = tc_smem(reinterpret_cast<uint8_t*>(bars) + 464);
            uint32_t dst, rbar0;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(dst) : "r"(src - 16), "r"(0));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbar0) : "r"(conv(0)), "r"(0));
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kS;
                const uint32_t ph = (uint32_t)((kb / kS) & 1);
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
        // ---------------- split pass, then epilogue (warps 2..17) ----------------
        // Two groups of 8 warps take alternate K blocks, so two blocks' splits
        // are in flight at once: one warp's per-block sequence (loads, convert,
        // TMEM / smem stores, wait::st, fences, barrier round trips) is longer
        // than the MMAs of a block, and with every warp on every block the
        // split pass, not the tensor pipe, set the pace.  Within a group a
        // thread converts one A row and one B column, 16 K values each.
        constexpr int kWpg = kH3SplitWarps / kH3Groups;  // warps per group (4 or 8)
        constexpr int kHalves = 8 / kWpg;                // K halves per thread and block (2 or 1)
        const int grp = (warp - 2) / kWpg;               // this group takes K blocks grp, grp + kH3Groups, ...
        const int w8 = (warp - 2) % kWpg;
        const int quarter = warp & 3;              // TMEM lanes this warp may access
        const int r = quarter * 32 + lane;         // A row of the tile / B column of this CTA's half
        const int khalf0 = w8 >> 2;                // first K half [16 khalf, +16) of the block
        const int ma = m0 + r, nb = nbl + r;
        const int ea = ma < args.M ? h3_exp(args.amax[ma]) : 0;
        const int eb = nb < args.N ? h3_exp(args.bmax[nb]) : 0;
        const float sa = h3_pow2(14 - ea), sb = h3_pow2(14 - eb);
        for (int kb = grp; kb < nkb; kb += kH3Groups) {
            const int l = kb % kL, s = kb % kS;
            tc_mbar_wait(full(l), (uint32_t)((kb / kL) & 1));
            float v[16];
            uint32_t ahi[kHalves][8], alo[kHalves][8], bhi[kHalves][8], blo[kHalves][8];
#pragma unroll
            for (int h = 0; h < kHalves; ++h) {
                const int khalf = khalf0 + h;
                if (args.diag & 1) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) ahi[h][j] = alo[h][j] = bhi[h][j] = blo[h][j] = 0u;
                } else {
                    if (args.diag & 64) {  // experiment: the conversions without the landing-tile reads
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __int_as_float(0x3f800000 + kb * 16 + j + lane);
                    } else {
                        h3_load16<A_MN>(landA(l), r, khalf, v);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) h3_split2(v[2 * j], v[2 * j + 1], sa, ahi[h][j], alo[h][j]);
                    if (args.diag & 64) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __int_as_float(0x3f000000 + kb * 16 + j + lane);
                    } else {
                        h3_load16<B_MN>(landB(l), r, khalf, v);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) h3_split2(v[2 * j], v[2 * j + 1], sb, bhi[h][j], blo[h][j]);
                }
            }
            // landing slot read (the values are consumed above): release it
            __syncwarp();
            if (lane == 0) tc_mbar_arrive(lempty(l));
            // f16 slot s free once the MMAs of K block kb - kS have completed
            tc_mbar_wait(fempty(s), (uint32_t)(((kb / kS) & 1) ^ 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int h = 0; h < kHalves; ++h) {
                const int khalf = khalf0 + h;
                const uint32_t tA =
                    tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(Cfg::kBN + 32 * s + 8 * khalf);
                if (!(args.diag & 16)) {
                    h3_st8(tA, ahi[h]);
                    h3_st8(tA + 16u, alo[h]);
                }
                // this thread's B column in the no-swizzle K-major f16 tiles: row r
                // of 8-row group r/8, K core matrices 2 khalf, 2 khalf + 1
                const uint32_t bh = tileBh(s) + (uint32_t)((r >> 3) * 512 + (2 * khalf) * 128 + (r & 7) * 16);
                if (!(args.diag & 32)) {
                    h3_sts4(bh, bhi[h][0], bhi[h][1], bhi[h][2], bhi[h][3]);
                    h3_sts4(bh + 128, bhi[h][4], bhi[h][5], bhi[h][6], bhi[h][7]);
                    h3_sts4(bh + Cfg::kB16, blo[h][0], blo[h][1], blo[h][2], blo[h][3]);
                    h3_sts4(bh + Cfg::kB16 + 128, blo[h][4], blo[h][5], blo[h][6], blo[h][7]);
                }
            }
            if (!(args.diag & 32)) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            if (!(args.diag & 16)) asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (PAIR && rank == 0 && w8 == 0)
                    tc_mbar_expect_tx(conv(s), 16);  // rank 1's forward (16-byte bulk copy)
                else
                    tc_mbar_arrive(conv(s));
            }
        }
        tc_mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int m = ma;
        const float ia = h3_pow2(ea - 14);
        constexpr int kCols = Cfg::kBN / (kH3SplitWarps / 4);  // columns per warp
        const int cbeg = ((warp - 2) >> 2) * kCols;
        // optional maxima of the output operand the next GEMMs consume (tanh(z)
        // for BIAS_TANH, C otherwise): per row (atomicMax once per thread) and
        // per column (warp max over this warp's 32 rows, one atomicMax per lane)
        const bool omax = args.omax_row != nullptr && !split && tail < 0;
        unsigned rmax = 0;
        // this warp's store staging (C, then C2): 8 KB of the landing ring,
        // idle once every K block has been split -- or, for the dgrad, whose
        // activations the producer prefetches into the landing ring, 4 KB of
        // the f16 ring (idle once every MMA has completed)
        const bool aux_smem = E == TcEpi::TANH_GRAD && PAIR && !split && tail < 0;
        const uint32_t stg = aux_smem ? f16base + (uint32_t)((warp - 2) * 4096) : sbase + (uint32_t)((warp - 2) * 8192);
        uint32_t aux_base = 0;  // this warp's activations: [column half][row quarter] 4 KB boxes
        if (aux_smem) {
            const int kb = nkb + ((warp - 2) >> 2);
            tc_mbar_wait(full(kb % kL), (uint32_t)((kb / kL) & 1));
            aux_base = landA(kb % kL) + (uint32_t)(quarter * 4096);
        }
        bool stg_pending = false;
#pragma unroll 1
        for (int c0 = cbeg; c0 < cbeg + kCols; c0 += 32) {
            uint32_t rr[32];
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]),
                  "=r"(rr[7]), "=r"(rr[8]), "=r"(rr[9]), "=r"(rr[10]), "=r"(rr[11]), "=r"(rr[12]), "=r"(rr[13]),
                  "=r"(rr[14]), "=r"(rr[15]), "=r"(rr[16]), "=r"(rr[17]), "=r"(rr[18]), "=r"(rr[19]),
                  "=r"(rr[20]), "=r"(rr[21]), "=r"(rr[22]), "=r"(rr[23]), "=r"(rr[24]), "=r"(rr[25]),
                  "=r"(rr[26]), "=r"(rr[27]), "=r"(rr[28]), "=r"(rr[29]), "=r"(rr[30]), "=r"(rr[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            const int nb0 = n0 + c0;
            if (nb0 >= args.N) continue;  // warp-uniform
            // undo the operand scales: two exact power-of-two products
            float x[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const int n = nb0 + q;
                const float ib = n < args.N ? h3_pow2(h3_exp(__ldg(args.bmax + n)) - 14) : 0.0f;
                x[q] = (__uint_as_float(rr[q]) * ia) * ib;
            }
            const bool mrow = m < args.M;
            if (tail >= 0) {
                // raw (scales undone) partial of this K half, tile-local [256][256]
                float* P = args.tail_part + (size_t)tail * (2 * kTcBM * Cfg::kBN) +
                           (size_t)(m - mt * 2 * kTcBM) * Cfg::kBN + c0;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    reinterpret_cast<float4*>(P)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
                continue;
            }
            if (split) {
                if (mrow) {
                    float* P = args.part + (size_t)blockIdx.z * args.M * args.N + (size_t)m * args.N;
                    if (nb0 + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            reinterpret_cast<float4*>(P + nb0)[q] =
                                make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
                    } else {
                        for (int q = 0; q < 32; ++q)
                            if (nb0 + q < args.N) P[nb0 + q] = x[q];
                    }
                }
                continue;
            }
            uint32_t ob[32];  // |consumed output| bits (0 past M / N)
            float cv[32], c2v[32];  // the chunk's C and (BIAS_TANH) C2 values of this row
            if (nb0 + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float4 vv = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
                    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (aux_smem) {
                        if constexpr (E == TcEpi::TANH_GRAD) {
                            float4 a;
                            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                                         : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                                         : "r"(aux_base + (uint32_t)(((c0 >> 5) & 1) * 16384 + lane * 128 +
                                                                     ((q ^ (lane & 7)) * 16))));
                            vv.x = tanh_grad(a.x, vv.x);
                            vv.y = tanh_grad(a.y, vv.y);
                            vv.z = tanh_grad(a.z, vv.z);
                            vv.w = tanh_grad(a.w, vv.w);
                        }
                    } else if (mrow) {
                        vv = tc_epi4<E>(args, m, nb0 + 4 * q, vv, &t);
                    }
                    cv[4 * q + 0] = vv.x;
                    cv[4 * q + 1] = vv.y;
                    cv[4 * q + 2] = vv.z;
                    cv[4 * q + 3] = vv.w;
                    c2v[4 * q + 0] = t.x;
                    c2v[4 * q + 1] = t.y;
                    c2v[4 * q + 2] = t.z;
                    c2v[4 * q + 3] = t.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int n = nb0 + q;
                    float vv = x[q], o2 = 0.0f;
                    if (n < args.N && mrow) {
                        const size_t idx = (size_t)m * args.N + n;
                        if constexpr (E == TcEpi::BIAS || E == TcEpi::BIAS_TANH) vv = sadd(vv, args.bias[n]);
                        if constexpr (E == TcEpi::TANH_GRAD) vv = tanh_grad(args.aux[idx], vv);
                        if constexpr (E == TcEpi::BIAS_TANH) o2 = tanhf(vv);
                        if constexpr (E == TcEpi::STORE)
                            if (args.out_scale != 0.0f) vv = smul(vv, args.out_scale);
                    }
                    cv[q] = vv;
                    c2v[q] = o2;
                }
            }
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const float o = E == TcEpi::BIAS_TANH ? c2v[q] : cv[q];
                ob[q] = (mrow && nb0 + q < args.N) ? __float_as_uint(fabsf(o)) : 0u;
            }
            // Stores: the warp stages its 32 rows x 32 columns in the (now idle)
            // landing ring, row-major with the 128-byte swizzle, and one lane
            // TMA-stores the box -- full-line writes (the tensor map clips rows
            // and columns past M and N).  Row-per-thread float4 stores touched 32
            // lines per instruction and cost 53 us of the 4096^3 forward's 350.
            if (!(args.diag & 128)) {
                if (lane == 0 && stg_pending) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t off = (uint32_t)(lane * 128 + ((q ^ (lane & 7)) * 16));
                    h3_sts4(stg + off, __float_as_uint(cv[4 * q]), __float_as_uint(cv[4 * q + 1]),
                            __float_as_uint(cv[4 * q + 2]), __float_as_uint(cv[4 * q + 3]));
                    if constexpr (E == TcEpi::BIAS_TANH)
                        h3_sts4(stg + 4096 + off, __float_as_uint(c2v[4 * q]), __float_as_uint(c2v[4 * q + 1]),
                                __float_as_uint(c2v[4 * q + 2]), __float_as_uint(c2v[4 * q + 3]));
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    const int mrow0 = m0 + quarter * 32;
                    h3_tma_store_2d(&tmC, stg, nb0, mrow0);
                    if constexpr (E == TcEpi::BIAS_TANH) h3_tma_store_2d(&tmC2, stg + 4096, nb0, mrow0);
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
                stg_pending = true;
            }
            if (omax) {
                unsigned mine = 0;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    rmax = max(rmax, ob[q]);
                    const unsigned cm = __reduce_max_sync(0xffffffffu, ob[q]);
                    if (lane == q) mine = cm;
                }
                if (nb0 + lane < args.N) atomicMax(args.omax_col + nb0 + lane, mine);
            }
        }
        if (omax && m < args.M) atomicMax(args.omax_row + m, rmax);
        if (lane == 0 && stg_pending) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
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

// ---- operand maxima (the scales' source) -------------------------------------
// max |x| of every row of a row-major R x C matrix (C % 4 == 0), as float bits
// (non-negative floats order like their bit patterns).  One warp per row.
__global__ void __launch_bounds__(256) k_absmax_rows(const float* __restrict__ X, int R, int C, unsigned* out) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= R) return;
    const float4* x = reinterpret_cast<const float4*>(X + (size_t)row * C);
    unsigned m = 0;
    for (int q = lane; q < C / 4; q += 32) {
        const float4 v = __ldg(x + q);
        m = max(m, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                       max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) out[row] = m;
}

// max |x| of every column (out zeroed beforehand): thread = 4 columns x a chunk
// of rows, one atomicMax per column per chunk
constexpr int kAbsmaxRows = 64;
__global__ void __launch_bounds__(256) k_absmax_cols(const float* __restrict__ X, int R, int C, unsigned* out) {
    const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * c4 >= C) return;
    const int r0 = blockIdx.y * kAbsmaxRows, r1 = min(R, r0 + kAbsmaxRows);
    unsigned m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    for (int r = r0; r < r1; ++r) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + (size_t)r * C) + c4);
        m0 = max(m0, __float_as_uint(fabsf(v.x)));
        m1 = max(m1, __float_as_uint(fabsf(v.y)));
        m2 = max(m2, __float_as_uint(fabsf(v.z)));
        m3 = max(m3, __float_as_uint(fabsf(v.w)));
    }
    atomicMax(out + 4 * c4 + 0, m0);
    atomicMax(out + 4 * c4 + 1, m1);
    atomicMax(out + 4 * c4 + 2, m2);
    atomicMax(out + 4 * c4 + 3, m3);
}

// max |x| of every row AND every column of a row-major R x C matrix in one
// pass (both zeroed beforehand): thread = 4 columns x kAbsmaxRows rows, rows
// loaded 8 at a time (memory-level parallelism); a row's partial over the
// warp's 128 columns is one redux, the block's 8 warps meet in shared memory
// and one atomicMax per row and block goes out (8x fewer same-address
// atomics than one per warp; C5: 167 -> 159 us per step for 10 matrices)
__global__ void __launch_bounds__(256) k_absmax_rc(const float* __restrict__ X, int R, int C, unsigned* rows,
                                                   unsigned* cols) {
    __shared__ unsigned rmax[8][kAbsmaxRows];
    const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5;
    const bool on = 4 * c4 < C;
    const int r0 = blockIdx.y * kAbsmaxRows, r1 = min(R, r0 + kAbsmaxRows);
    unsigned m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    for (int rb = r0; rb < r0 + kAbsmaxRows; rb += 8) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            v[j] = (on && rb + j < r1) ? __ldg(reinterpret_cast<const float4*>(X + (size_t)(rb + j) * C) + c4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned a = __float_as_uint(fabsf(v[j].x)), b = __float_as_uint(fabsf(v[j].y));
            const unsigned c = __float_as_uint(fabsf(v[j].z)), d = __float_as_uint(fabsf(v[j].w));
            m0 = max(m0, a);
            m1 = max(m1, b);
            m2 = max(m2, c);
            m3 = max(m3, d);
            const unsigned rm = __reduce_max_sync(0xffffffffu, max(max(a, b), max(c, d)));
            if ((threadIdx.x & 31) == j) rmax[warp][rb + j - r0] = rm;
        }
    }
    __syncthreads();
    if (threadIdx.x < kAbsmaxRows && r0 + (int)threadIdx.x < r1) {
        unsigned rm = rmax[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < 8; ++w) rm = max(rm, rmax[w][threadIdx.x]);
        if (rm) atomicMax(rows + r0 + threadIdx.x, rm);
    }
    if (on) {
        atomicMax(cols + 4 * c4 + 0, m0);
        atomicMax(cols + 4 * c4 + 1, m1);
        atomicMax(cols + 4 * c4 + 2, m2);
        atomicMax(cols + 4 * c4 + 3, m3);
    }
}


// Finish the tail-wave tiles: sum the two K halves (half 0 + half 1, fixed
// order), then the epilogue and the optional output maxima.  Grid (tail tiles,
// 16 chunks of 16 rows), 256 threads: 64 float4 columns x 4 row lanes, each
// thread 4 rows (8 independent float4 loads in flight).  The first version
// (one column per thread, a 32-row loop of scalar loads) took ~19 us per
// GEMM at C5 -- 5% of the step.
constexpr int kTailRows = 16;
template <TcEpi E>
__global__ void __launch_bounds__(256) k_h3_tail_reduce(TcArgs a) {
    const int t = a.full_units + (int)blockIdx.x;
    int mt, nt;
    h3_tile_mn(t, a.tiles_m, a.tiles_n, mt, nt);
    const int c4 = (int)threadIdx.x & 63, ry = (int)threadIdx.x >> 6;
    const int n = nt * 256 + 4 * c4;
    const bool ncol = n < a.N;  // N % 4 == 0: the float4 is in or out as a whole
    const float* P0 = a.tail_part + (size_t)(2 * blockIdx.x) * 65536;
    const float* P1 = P0 + 65536;
    float4 v0[4], v1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int lr = (int)blockIdx.y * kTailRows + ry + 4 * i;
        v0[i] = *reinterpret_cast<const float4*>(P0 + lr * 256 + 4 * c4);
        v1[i] = *reinterpret_cast<const float4*>(P1 + lr * 256 + 4 * c4);
    }
    unsigned cm[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int lr = (int)blockIdx.y * kTailRows + ry + 4 * i;
        const int m = mt * 256 + lr;
        unsigned ob[4] = {0u, 0u, 0u, 0u};
        if (m < a.M && ncol) {
            float4 v = make_float4(v0[i].x + v1[i].x, v0[i].y + v1[i].y, v0[i].z + v1[i].z, v0[i].w + v1[i].w);
            float4 o2 = make_float4(0.f, 0.f, 0.f, 0.f);
            v = tc_epi4<E>(a, m, n, v, &o2);
            const size_t idx = (size_t)m * a.N + n;
            *reinterpret_cast<float4*>(a.C + idx) = v;
            if constexpr (E == TcEpi::BIAS_TANH) *reinterpret_cast<float4*>(a.C2 + idx) = o2;
            const float4 o = E == TcEpi::BIAS_TANH ? o2 : v;
            ob[0] = __float_as_uint(fabsf(o.x));
            ob[1] = __float_as_uint(fabsf(o.y));
            ob[2] = __float_as_uint(fabsf(o.z));
            ob[3] = __float_as_uint(fabsf(o.w));
        }
        if (a.omax_row) {
#pragma unroll
            for (int j = 0; j < 4; ++j) cm[j] = max(cm[j], ob[j]);
            const unsigned rm = __reduce_max_sync(0xffffffffu, max(max(ob[0], ob[1]), max(ob[2], ob[3])));
            if ((threadIdx.x & 31) == 0 && m < a.M && rm) atomicMax(a.omax_row + m, rm);
        }
    }
    if (a.omax_row) {
        // column maxima over the block's 16 rows: the 4 row lanes through shared memory
        __shared__ unsigned sc[4][256];
#pragma unroll
        for (int j = 0; j < 4; ++j) sc[ry][4 * c4 + j] = cm[j];
        __syncthreads();
        const int col = (int)threadIdx.x;
        const unsigned v = max(max(sc[0][col], sc[1][col]), max(sc[2][col], sc[3][col]));
        if (nt * 256 + col < a.N && v) atomicMax(a.omax_col + nt * 256 + col, v);
    }
}

}  // namespace lane_b200

// ---------------------------------------------------------------- host side
namespace lane_b200 {

// row and column maxima of a row-major R x C matrix (C % 4 == 0) into zeroed
// `rows` / `cols`
inline void absmax_rc_launch(cudaStream_t st, const float* X, int R, int C, unsigned* rows, unsigned* cols) {
    k_absmax_rc<<<dim3((unsigned)((C / 4 + 255) / 256), (unsigned)((R + kAbsmaxRows - 1) / kAbsmaxRows)), 256, 0,
                  st>>>(X, R, C, rows, cols);
}

// maxima of the rows (rows = true) or columns of a row-major R x C matrix
inline void absmax_launch(cudaStream_t st, const float* X, int R, int C, bool rows, unsigned* out) {
    if (rows) {
        k_absmax_rows<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(X, R, C, out);
    } else {
        LANE_CUDA(cudaMemsetAsync(out, 0, (size_t)C * sizeof(unsigned), st));
        k_absmax_cols<<<dim3((unsigned)((C / 4 + 255) / 256), (unsigned)((R + kAbsmaxRows - 1) / kAbsmaxRows)), 256,
                        0, st>>>(X, R, C, out);
    }
}

template <bool A_MN, bool B_MN, TcEpi E, bool PAIR>
inline void h3_launch(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                      const CUtensorMap& c2, const TcArgs& args) {
    constexpr size_t smem = H3Cfg<PAIR>::kSmem;
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    LANE_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        LANE_CUDA(cudaFuncSetAttribute(k_gemm_h3<A_MN, B_MN, E, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        configured.fetch_or(bit, std::memory_order_release);
    }
    const int S = args.kbs > 0 ? (args.K / kTcBK + args.kbs - 1) / args.kbs : 1;
    if constexpr (PAIR) {
        cudaLaunchConfig_t cfg = {};
        constexpr int kBN = H3Cfg<true>::kBN;
        cfg.gridDim = dim3(2 * ((args.M + 2 * kTcBM - 1) / (2 * kTcBM)), (args.N + kBN - 1) / kBN, S);
        if (args.full_units > 0)  // tail-wave split: whole tiles, then two K halves per tail tile
            cfg.gridDim = dim3(2 * (args.full_units + 2 * (args.tiles_m * args.tiles_n - args.full_units)), 1, 1);
        cfg.blockDim = dim3(kH3Threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LANE_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_h3<A_MN, B_MN, E, PAIR>, a, b, c, c2, args));
    } else {
        const dim3 grid((args.N + kTcBN - 1) / kTcBN, (args.M + kTcBM - 1) / kTcBM, S);
        k_gemm_h3<A_MN, B_MN, E, PAIR><<<grid, kH3Threads, smem, st>>>(a, b, c, c2, args);
    }
    if (S > 1) {
        const size_t n4 = (size_t)args.M * args.N / 4;
        k_tc_splitk_reduce<E><<<(unsigned)std::min<size_t>(1184, (n4 + 255) / 256), 256, 0, st>>>(args, S);
    }
    if (PAIR && args.full_units > 0)
        k_h3_tail_reduce<E><<<dim3((unsigned)(args.tiles_m * args.tiles_n - args.full_units), 256 / kTailRows), 256, 0,
                              st>>>(args);
}

template <TcEpi E, bool PAIR>
inline void h3_dispatch(cudaStream_t st, bool a_mn, bool b_mn, const CUtensorMap& a, const CUtensorMap& b,
                        const CUtensorMap& c, const CUtensorMap& c2, const TcArgs& args) {
    if (!a_mn && !b_mn) h3_launch<false, false, E, PAIR>(st, a, b, c, c2, args);
    else if (!a_mn && b_mn) h3_launch<false, true, E, PAIR>(st, a, b, c, c2, args);
    else if (a_mn && !b_mn) h3_launch<true, false, E, PAIR>(st, a, b, c, c2, args);
    else h3_launch<true, true, E, PAIR>(st, a, b, c, c2, args);
}

}  // namespace lane_b200
