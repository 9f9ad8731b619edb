// gemm.cuh -- fp32 GEMMs of the mini-batch path with fused epilogues.
//
// Three operand layouts cover the whole step (row-major everywhere):
//   NN  C[M,N] = A[M,K]   B[K,N]      forward   Z = X W
//   NT  C[M,N] = A[M,K]   B[N,K]^T    dgrad     S = D' W'^T  (W' is O x O')
//   TN  C[M,N] = A[K,M]^T B[K,N]      wgrad     G = X^T D
// Epilogues: STORE, BIAS (+b[n]), BIAS_TANH (z and tanh(z)), TANH_GRAD
// ((1 - a^2) * acc with a = aux[m,n]).
//
// This file holds the SIMT (CUDA-core FFMA) kernel: exact fp32 products with
// fp32 accumulation, 128x128x8 tiles, 8x8 outputs per thread, double-buffered
// shared memory.  gemm() dispatches large GEMMs to the tcgen05 3xTF32 kernel
// (gemm_tc.cuh) when it is enabled and the shape qualifies.
#pragma once

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "gemm_tcp.cuh"
#include "gemm_h3.cuh"

namespace lane_b200 {

enum class GemmOp { NN, NT, TN };
enum class Epi { STORE, BIAS, BIAS_TANH, TANH_GRAD };

struct GemmCtx {
    cudaStream_t stream;
    int sm_count;
    float** ws;
    size_t* ws_count;
    uint64_t* launches;
    uint64_t* ws_gen = nullptr;  // bumped on every reallocation (captured graphs key on it)
    int** counters = nullptr;    // stream-K tile arrival counters (zero between launches)
    size_t* counters_count = nullptr;
};

// 3xF16 operand maxima supplied by the caller (gemm_h3.cuh): a = rows of
// op(A), b = columns of op(B); orow / ocol (zeroed by the caller) receive the
// row / column maxima of the output operand the next GEMMs read (tanh(z) for
// BIAS_TANH, C otherwise) -- fused into the 3xF16 epilogue, or one extra pass
// when the GEMM runs another kernel.
struct GemmMax {
    const unsigned* a = nullptr;
    const unsigned* b = nullptr;
    unsigned* orow = nullptr;
    unsigned* ocol = nullptr;
    float out_scale = 0.0f;  // STORE on the 3xF16 kernel: C = sum * out_scale (0: none)
};

inline void ensure_ws(GemmCtx& g, size_t count) {
    if (*g.ws_count >= count) return;
    if (*g.ws) LANE_CUDA(cudaFree(*g.ws));
    LANE_CUDA(cudaMalloc(reinterpret_cast<void**>(g.ws), count * sizeof(float)));
    *g.ws_count = count;
    if (g.ws_gen) ++*g.ws_gen;
}

// stream-K arrival counters: zeroed once at allocation, reset to zero by the
// kernel's last arriving piece of every tile
inline bool ensure_counters(GemmCtx& g, size_t count) {
    if (!g.counters || !g.counters_count) return false;
    if (*g.counters_count >= count) return true;
    if (*g.counters) LANE_CUDA(cudaFree(*g.counters));
    LANE_CUDA(cudaMalloc(reinterpret_cast<void**>(g.counters), count * sizeof(int)));
    LANE_CUDA(cudaMemsetAsync(*g.counters, 0, count * sizeof(int), g.stream));
    *g.counters_count = count;
    if (g.ws_gen) ++*g.ws_gen;
    return true;
}

template <Epi E>
__device__ __forceinline__ void epilogue_store(int m, int n, int N, float acc, float* C, float* C2,
                                               const float* bias, const float* aux) {
    const size_t idx = (size_t)m * N + n;
    if constexpr (E == Epi::STORE) {
        C[idx] = acc;
    } else if constexpr (E == Epi::BIAS) {
        C[idx] = sadd(acc, bias[n]);
    } else if constexpr (E == Epi::BIAS_TANH) {
        const float z = sadd(acc, bias[n]);
        C[idx] = z;
        C2[idx] = tanhf(z);
    } else {
        C[idx] = tanh_grad(aux[idx], acc);
    }
}

constexpr int kBM = 128, kBN = 128, kBK = 8;

template <GemmOp OP, Epi E>
__global__ void __launch_bounds__(256) k_gemm_simt(int M, int N, int K, const float* __restrict__ A,
                                                   int lda, const float* __restrict__ B, int ldb,
                                                   float* __restrict__ C, float* __restrict__ C2,
                                                   const float* __restrict__ bias,
                                                   const float* __restrict__ aux) {
    __shared__ __align__(16) float As[2][kBK][kBM];
    __shared__ __align__(16) float Bs[2][kBK][kBN];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
    const int tx = tid % 16, ty = tid / 16;

    float a_reg[4], b_reg[4];
    auto load_tiles = [&](int k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if constexpr (OP == GemmOp::TN) {
                // A[k*lda + m]: k = tid/32, m = (tid%32)*4 + u
                const int k = k0 + tid / 32, m = m0 + (tid % 32) * 4 + u;
                a_reg[u] = (k < K && m < M) ? A[(size_t)k * lda + m] : 0.0f;
            } else {
                // A[m*lda + k]: m = tid/2, k = (tid%2)*4 + u
                const int m = m0 + tid / 2, k = k0 + (tid % 2) * 4 + u;
                a_reg[u] = (k < K && m < M) ? A[(size_t)m * lda + k] : 0.0f;
            }
            if constexpr (OP == GemmOp::NT) {
                // B[n*ldb + k]: n = tid/2, k = (tid%2)*4 + u
                const int n = n0 + tid / 2, k = k0 + (tid % 2) * 4 + u;
                b_reg[u] = (k < K && n < N) ? B[(size_t)n * ldb + k] : 0.0f;
            } else {
                // B[k*ldb + n]: k = tid/32, n = (tid%32)*4 + u
                const int k = k0 + tid / 32, n = n0 + (tid % 32) * 4 + u;
                b_reg[u] = (k < K && n < N) ? B[(size_t)k * ldb + n] : 0.0f;
            }
        }
    };
    auto store_tiles = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if constexpr (OP == GemmOp::TN) As[buf][tid / 32][(tid % 32) * 4 + u] = a_reg[u];
            else As[buf][(tid % 2) * 4 + u][tid / 2] = a_reg[u];
            if constexpr (OP == GemmOp::NT) Bs[buf][(tid % 2) * 4 + u][tid / 2] = b_reg[u];
            else Bs[buf][tid / 32][(tid % 32) * 4 + u] = b_reg[u];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

    load_tiles(0);
    store_tiles(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += kBK) {
        const bool more = k0 + kBK < K;
        if (more) load_tiles(k0 + kBK);
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) {
            store_tiles(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (n < N) epilogue_store<E>(m, n, N, acc[i][j], C, C2, bias, aux);
        }
    }
}

template <GemmOp OP>
void gemm_simt_dispatch(GemmCtx& g, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                        Epi e, float* C, float* C2, const float* bias, const float* aux) {
    const dim3 grid((N + kBN - 1) / kBN, (M + kBM - 1) / kBM);
    switch (e) {
        case Epi::STORE:
            k_gemm_simt<OP, Epi::STORE><<<grid, 256, 0, g.stream>>>(M, N, K, A, lda, B, ldb, C, C2, bias, aux);
            break;
        case Epi::BIAS:
            k_gemm_simt<OP, Epi::BIAS><<<grid, 256, 0, g.stream>>>(M, N, K, A, lda, B, ldb, C, C2, bias, aux);
            break;
        case Epi::BIAS_TANH:
            k_gemm_simt<OP, Epi::BIAS_TANH><<<grid, 256, 0, g.stream>>>(M, N, K, A, lda, B, ldb, C, C2, bias,
                                                                         aux);
            break;
        case Epi::TANH_GRAD:
            k_gemm_simt<OP, Epi::TANH_GRAD><<<grid, 256, 0, g.stream>>>(M, N, K, A, lda, B, ldb, C, C2, bias,
                                                                         aux);
            break;
    }
    *g.launches += 1;
}

// ---- skinny GEMMs (N <= 32: the 10-class output layer) --------------------
// NN: C[M,N] = A[M,K] B[K,N].  A CTA of kSkNW warps owns one row m; warp w
// takes the K range [w K/kSkNW, (w+1) K/kSkNW) with lanes striding it
// (coalesced A row), N partial sums per lane in registers; shuffle reduction
// per warp, then the kSkNW warp sums in a fixed order (deterministic).
constexpr int kSkNW = 4;
template <Epi E>
__global__ void __launch_bounds__(32 * kSkNW) k_gemm_skinny_nn(int M, int N, int K, const float* __restrict__ A,
                                                               const float* __restrict__ B, float* __restrict__ C,
                                                               float* __restrict__ C2, const float* __restrict__ bias) {
    __shared__ float part[kSkNW][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = warp * K / kSkNW, k1 = (warp + 1) * K / kSkNW;
    for (int m = blockIdx.x; m < M; m += gridDim.x) {
        float acc[32];
#pragma unroll
        for (int n = 0; n < 32; ++n) acc[n] = 0.0f;
        const float* arow = A + (size_t)m * K;
#pragma unroll 4
        for (int k = k0 + lane; k < k1; k += 32) {
            const float a = __ldg(arow + k);
            const float* brow = B + (size_t)k * N;
#pragma unroll
            for (int n = 0; n < 32; ++n)
                if (n < N) acc[n] = fmaf(a, __ldg(brow + n), acc[n]);
        }
#pragma unroll
        for (int n = 0; n < 32; ++n)
            if (n < N) acc[n] = warp_sum(acc[n]);
        if (lane == 0) {
#pragma unroll
            for (int n = 0; n < 32; ++n)
                if (n < N) part[warp][n] = acc[n];
        }
        __syncthreads();
        if (threadIdx.x < N) {
            const int n = threadIdx.x;
            float v = part[0][n];
#pragma unroll
            for (int w = 1; w < kSkNW; ++w) v += part[w][n];
            const size_t idx = (size_t)m * N + n;
            if constexpr (E == Epi::BIAS || E == Epi::BIAS_TANH) v = sadd(v, bias[n]);
            C[idx] = v;
            if constexpr (E == Epi::BIAS_TANH) C2[idx] = tanhf(v);
        }
        __syncthreads();
    }
}

// TN: C[M,N] = A^T B with A [K][M] (lda = M), B [K][N]; K is the batch.  A CTA
// owns 32 columns m x one K chunk of kSkinnyKChunk; its 4 warps split the
// chunk (warp w: k = k0 + w, k0 + w + 4, ...), lanes take consecutive m
// (coalesced A rows), N accumulators per thread; the 4 partials meet in
// shared memory (fixed order) and the per-chunk partial sums part[y][m][n]
// are reduced in a fixed order by k_sum_partials.
// dst[0..n) = src[0..n) with every load of the loop in flight together
// (float4 when src is 16-byte aligned; the serial load->store loop it replaces
// cost one L2 round trip per iteration)
__device__ __forceinline__ void stage_rows(float* dst, const float* __restrict__ src, int n) {
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const int n4 = n >> 2;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll 4
        for (int e = threadIdx.x; e < n4; e += blockDim.x) d4[e] = __ldg(s4 + e);
        for (int e = 4 * n4 + threadIdx.x; e < n; e += blockDim.x) dst[e] = __ldg(src + e);
    } else {
#pragma unroll 4
        for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = __ldg(src + e);
    }
}

constexpr int kSkinnyKChunk = 128;
constexpr int kSkTnW = 4;
// N <= NM (16 or 32): accumulators and the unrolled class loop; TW k-groups
// (warps) per CTA -- 8 for NM = 16, so more loads are in flight
template <int NM>
constexpr int skinny_tn_warps() { return NM == 16 ? 8 : kSkTnW; }
template <int NM>
__global__ void __launch_bounds__(32 * skinny_tn_warps<NM>()) k_gemm_skinny_tn(int M, int N, int K,
                                                                              const float* __restrict__ A,
                                                                              const float* __restrict__ B,
                                                                              float* __restrict__ part, int cpb) {
    constexpr int TW = skinny_tn_warps<NM>();
    // this CTA: K chunks [blockIdx.y * cpb, +cpb) (cpb = chunks per block)
    __shared__ __align__(16) float bs[kSkinnyKChunk * 32];
    __shared__ float red[TW][32][NM + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int m = blockIdx.x * 32 + tx;
    float acc[NM];
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = 0.0f;
    for (int c = 0; c < cpb; ++c) {
        const int k0 = (blockIdx.y * cpb + c) * kSkinnyKChunk, k1 = min(K, k0 + kSkinnyKChunk);
        if (k0 >= K) break;
        if (c) __syncthreads();
        stage_rows(bs, B + (size_t)k0 * N, (k1 - k0) * N);
        __syncthreads();
        if (m < M) {
#pragma unroll 4
            for (int k = k0 + ty; k < k1; k += TW) {
                const float a = __ldg(A + (size_t)k * M + m);
                const float* brow = bs + (k - k0) * N;
#pragma unroll
                for (int n = 0; n < NM; ++n)
                    if (n < N) acc[n] = fmaf(a, brow[n], acc[n]);
            }
        }
    }
#pragma unroll
    for (int n = 0; n < NM; ++n)
        if (n < N) red[ty][tx][n] = acc[n];
    __syncthreads();
    // thread (tx, ty): outputs n = ty, ty + TW, ... of column m
    if (m < M) {
        float* out = part + ((size_t)blockIdx.y * M + m) * N;
        for (int n = ty; n < N; n += TW) {
            float v = red[0][tx][n];
#pragma unroll
            for (int w = 1; w < TW; ++w) v += red[w][tx][n];
            out[n] = v;
        }
    }
}

// out[e] = sum_{s < S} part[s*count + e]  (fixed order: deterministic)
__global__ void k_sum_partials(const float* __restrict__ part, int S, size_t count, float* __restrict__ out) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
        float v = part[e];
        for (int s = 1; s < S; ++s) v += part[(size_t)s * count + e];
        out[e] = v;
    }
}

// Many partials (S >= 16): CTA = 32 consecutive elements x 8 partial groups
// (warp w sums partials w, w + 8, ... in order, lane = element), the 8 group
// sums meet in shared memory in a fixed order -- deterministic, and S / 8
// dependent loads per thread instead of S.
__global__ void __launch_bounds__(256) k_sum_partials_wide(const float* __restrict__ part, int S, size_t count,
                                                           float* __restrict__ out) {
    __shared__ float red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const size_t e = (size_t)blockIdx.x * 32 + lane;
    float v = 0.0f;
    if (e < count)
        for (int s = w; s < S; s += 8) v += __ldg(part + (size_t)s * count + e);
    red[w][lane] = v;
    __syncthreads();
    if (w == 0 && e < count) {
        float t = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; ++q) t += red[q][lane];
        out[e] = t;
    }
}

inline void sum_partials(GemmCtx& g, const float* part, int S, size_t count, float* out) {
    if (S >= 16)
        k_sum_partials_wide<<<(unsigned)((count + 31) / 32), 256, 0, g.stream>>>(part, S, count, out);
    else
        k_sum_partials<<<std::max(1, (int)std::min<size_t>(4 * g.sm_count, (count + 255) / 256)), 256, 0,
                         g.stream>>>(part, S, count, out);
}

// Column sums gb[o] = sum_b D[b][o], two passes (row chunks, then fixed-order
// reduction) so tall batches keep every SM busy.
constexpr int kColChunk = 32;
__global__ void k_colsum_part(const float* __restrict__ D, int B, int O, float* __restrict__ part) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= O) return;
    const int b0 = blockIdx.y * kColChunk, b1 = min(B, b0 + kColChunk);
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // 4 independent chains: loads in flight
    int b = b0;
    for (; b + 4 <= b1; b += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] += __ldg(D + (size_t)(b + u) * O + o);
    }
    for (; b < b1; ++b) v[0] += __ldg(D + (size_t)b * O + o);
    part[(size_t)blockIdx.y * O + o] = (v[0] + v[1]) + (v[2] + v[3]);
}

// One pass: CTA = 32 columns x 16 row groups (warp w sums rows b = w mod 16,
// eight independent chains so a warp keeps eight loads in flight), the 16
// group sums meet in shared memory in a fixed order.
__global__ void __launch_bounds__(512) k_colsum(const float* __restrict__ D, int B, int O, float* __restrict__ gb) {
    __shared__ float red[16][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int o = blockIdx.x * 32 + lane;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (o < O) {
        int b = w;
        for (; b + 7 * 16 < B; b += 8 * 16) {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] += __ldg(D + (size_t)(b + 16 * u) * O + o);
        }
        for (; b < B; b += 16) v[0] += __ldg(D + (size_t)b * O + o);
    }
    red[w][lane] = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    __syncthreads();
    if (w == 0 && o < O) {
        float t = red[0][lane];
#pragma unroll
        for (int q = 1; q < 16; ++q) t += red[q][lane];
        gb[o] = t;
    }
}

inline void colsum(GemmCtx& g, const float* D, int B, int O, float* gb) {
    if (B <= 1024 && ((O + 31) / 32 >= g.sm_count / 2 || B <= 256)) {
        k_colsum<<<(O + 31) / 32, 512, 0, g.stream>>>(D, B, O, gb);
        *g.launches += 1;
        return;
    }
    // narrow and tall: row chunks first so every SM streams, then a fixed-order sum
    const int S = (B + kColChunk - 1) / kColChunk;
    ensure_ws(g, (size_t)S * O);
    k_colsum_part<<<dim3((O + 127) / 128, S), 128, 0, g.stream>>>(D, B, O, *g.ws);
    sum_partials(g, *g.ws, S, (size_t)O, gb);
    *g.launches += 2;
}

// NN, K split into chunks with the B chunk staged in shared memory: CTA
// (row block of 8 rows, K chunk of kSkKC) -- warp w owns row m0+w, lanes
// stride the chunk (coalesced A row), N partial sums per lane, shuffle
// reduction; per-chunk partials part[y][m][n] are summed in a fixed order
// (with the epilogue) by k_sum_partials_epi.
constexpr int kSkKC = 512;
__global__ void __launch_bounds__(256) k_gemm_skinny_nn_kc(int M, int N, int K, const float* __restrict__ A,
                                                           const float* __restrict__ B, float* __restrict__ part,
                                                           int rpw) {
    __shared__ __align__(16) float bs[kSkKC * 16];
    const int k0 = blockIdx.y * kSkKC, k1 = min(K, k0 + kSkKC);
    stage_rows(bs, B + (size_t)k0 * N, (k1 - k0) * N);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // rpw rows per warp (up to 8 when the rows are many), so a staged B chunk
    // serves more rows (C5: 16 MB of B staging instead of 128 MB for 64 MB of A)
#pragma unroll 1
    for (int rr = 0; rr < rpw; ++rr) {
    const int m = (blockIdx.x * 8 + warp) * rpw + rr;
    if (m >= M) return;
    float acc[16];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n] = 0.0f;
    const float* arow = A + (size_t)m * K;
#pragma unroll 4
    for (int k = k0 + lane; k < k1; k += 32) {
        const float a = __ldg(arow + k);
        const float* brow = bs + (k - k0) * N;
#pragma unroll
        for (int n = 0; n < 16; ++n)
            if (n < N) acc[n] = fmaf(a, brow[n], acc[n]);
    }
    // transpose-reduce the 16 sums over the warp (fixed butterfly, 16
    // shuffles instead of 16 x 5): after the offsets 16, 8, 4, 2 a lane holds
    // the partial of value idx = its lane bits 4..1; offset 1 completes it
    int nv = 16;
#pragma unroll
    for (int o = 16; o >= 2; o >>= 1) {
        nv >>= 1;
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < nv) {
                const float send = hi ? acc[q] : acc[q + nv];
                const float keep = hi ? acc[q + nv] : acc[q];
                acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
    }
    const float v = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 1);
    const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
    if ((lane & 1) == 0 && idx < N) part[((size_t)blockIdx.y * M + m) * N + idx] = v;
    }
}

// Skinny NN, row per lane (M >= 2048, N <= 16, K % 4 == 0, 16-byte rows): the
// output layer's forward at C5 (4096 x 10 x 4096).  Block (256 rows, K chunk
// of kSrKC): lane = one row of A, which it streams as float4 along K -- the
// other half of each 32-byte sector is the next iteration's, an L1 hit -- and
// every B value is a broadcast shared-memory read (the whole warp reads the
// same k), so a k costs N / 4 broadcast LDS.128 for 32 x N FMAs and no
// cross-lane reduction.  The partials of the K chunks are summed in a fixed
// order with the epilogue (k_sum_partials_epi).  The lanes-along-K kernel
// above pays N conflicted LDS per k and lane: 68 us at C5 against 47 us here
// (the 64 MB read of A alone would take ~10 us; the 32-row loads are L1-
// wavefront bound).
constexpr int kSrKC = 128;
__global__ void __launch_bounds__(256) k_gemm_skinny_nn_rows(int M, int N, int K, const float* __restrict__ A,
                                                             const float* __restrict__ B, float* __restrict__ part) {
    __shared__ __align__(16) float bs[kSrKC * 16];  // [k][16], zero past N
    const int k0 = blockIdx.y * kSrKC, kn = min(K - k0, kSrKC);
    for (int e = threadIdx.x; e < kSrKC * 16; e += blockDim.x) {
        const int k = e >> 4, n = e & 15;
        bs[e] = (k < kn && n < N) ? __ldg(B + (size_t)(k0 + k) * N + n) : 0.0f;
    }
    __syncthreads();
    const int m = blockIdx.x * 256 + threadIdx.x;
    if (m >= M) return;
    const float4* arow = reinterpret_cast<const float4*>(A + (size_t)m * K + k0);
    const float4* b4 = reinterpret_cast<const float4*>(bs);
    float acc[16];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n] = 0.0f;
#pragma unroll 8
    for (int q = 0; q < kn / 4; ++q) {
        const float4 a = __ldg(arow + q);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 b = b4[(4 * q + j) * 4 + c];
                acc[4 * c + 0] = fmaf(av[j], b.x, acc[4 * c + 0]);
                acc[4 * c + 1] = fmaf(av[j], b.y, acc[4 * c + 1]);
                acc[4 * c + 2] = fmaf(av[j], b.z, acc[4 * c + 2]);
                acc[4 * c + 3] = fmaf(av[j], b.w, acc[4 * c + 3]);
            }
        }
    }
    float* out = part + ((size_t)blockIdx.y * M + m) * N;
#pragma unroll
    for (int n = 0; n < 16; ++n)
        if (n < N) out[n] = acc[n];
}

// out = epilogue(sum_{s < S} part[s]) in a fixed order; bias per column
template <Epi E>
__global__ void k_sum_partials_epi(const float* __restrict__ part, int S, int M, int N, float* __restrict__ C,
                                   float* __restrict__ C2, const float* __restrict__ bias) {
    const size_t count = (size_t)M * N;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
        float v = part[e];
        for (int s2 = 1; s2 < S; ++s2) v += part[(size_t)s2 * count + e];
        if constexpr (E == Epi::BIAS || E == Epi::BIAS_TANH) v = sadd(v, bias[(unsigned)e % (unsigned)N]);
        C[e] = v;
        if constexpr (E == Epi::BIAS_TANH) C2[e] = tanhf(v);
    }
}

// NT with a short K (the output layer's dgrad: D[M][K<=16] W[N][K]^T) and the
// tanh' epilogue: one thread per output column n holds W[n][:] in registers,
// 8 rows m per CTA (D rows broadcast from shared memory), sequential k.
constexpr int kShortK = 16;
template <Epi E>
__global__ void __launch_bounds__(256) k_gemm_shortk_nt(int M, int N, int K, const float* __restrict__ D,
                                                        const float* __restrict__ W, float* __restrict__ C,
                                                        const float* __restrict__ aux) {
    __shared__ float ds[8][kShortK];
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int m0 = blockIdx.y * 8;
    for (int e = threadIdx.x; e < 8 * K; e += blockDim.x) {
        const int r = e / K, k = e - r * K;
        ds[r][k] = m0 + r < M ? D[(size_t)(m0 + r) * K + k] : 0.0f;
    }
    __syncthreads();
    if (n >= N) return;
    float w[kShortK];
#pragma unroll
    for (int k = 0; k < kShortK; ++k) w[k] = k < K ? __ldg(W + (size_t)n * K + k) : 0.0f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int m = m0 + r;
        if (m >= M) break;
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < kShortK; ++k)
            if (k < K) acc = fmaf(ds[r][k], w[k], acc);
        const size_t idx = (size_t)m * N + n;
        if constexpr (E == Epi::TANH_GRAD) acc = tanh_grad(aux[idx], acc);
        C[idx] = acc;
    }
}

// The same for N % 4 == 0 and many rows (the C5 output layer's dgrad,
// 4096 x 4096 x 10): thread = 4 consecutive columns (float4 aux loads and C
// stores), CTA = 1024 columns x 32 rows, rows 4 at a time so four loads are
// in flight.  The plain kernel's 8-row CTAs re-read their W rows per CTA and
// moved 4 bytes per thread per row (1.7 TB/s).
constexpr int kShortRows = 32;  // rows per CTA at most (rows: a multiple of 4)
template <Epi E>
__global__ void __launch_bounds__(256) k_gemm_shortk_nt4(int M, int N, int K, const float* __restrict__ D,
                                                         const float* __restrict__ W, float* __restrict__ C,
                                                         const float* __restrict__ aux, int rows) {
    __shared__ float ds[kShortRows][kShortK];
    const int n4 = blockIdx.x * blockDim.x + threadIdx.x;  // columns 4 n4 .. 4 n4 + 3
    const int m0 = blockIdx.y * rows;
    for (int e = threadIdx.x; e < rows * kShortK; e += blockDim.x) {
        const int r = e / kShortK, k = e - r * kShortK;
        ds[r][k] = (m0 + r < M && k < K) ? D[(size_t)(m0 + r) * K + k] : 0.0f;
    }
    __syncthreads();
    if (4 * n4 >= N) return;
    float w[4][kShortK];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < kShortK; ++k) w[c][k] = k < K ? __ldg(W + (size_t)(4 * n4 + c) * K + k) : 0.0f;
#pragma unroll 1
    for (int r0 = 0; r0 < rows; r0 += 4) {
        float4 t[4];
        if constexpr (E == Epi::TANH_GRAD) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                t[q] = m0 + r0 + q < M ? __ldg(reinterpret_cast<const float4*>(aux + (size_t)(m0 + r0 + q) * N) + n4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = m0 + r0 + q;
            if (m >= M) break;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < kShortK; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] = fmaf(ds[r0 + q][k], w[c][k], acc[c]);
            float4 o = make_float4(acc[0], acc[1], acc[2], acc[3]);
            if constexpr (E == Epi::TANH_GRAD)
                o = make_float4(tanh_grad(t[q].x, acc[0]), tanh_grad(t[q].y, acc[1]), tanh_grad(t[q].z, acc[2]),
                                tanh_grad(t[q].w, acc[3]));
            reinterpret_cast<float4*>(C + (size_t)m * N)[n4] = o;
        }
    }
}

inline bool gemm_try_skinny(GemmCtx& g, GemmOp op, int M, int N, int K, const float* A, int lda, const float* B,
                            int ldb, Epi e, float* C, float* C2, const float* bias, const float* aux) {
    if (op == GemmOp::NT && K <= kShortK && lda == K && ldb == K && (e == Epi::STORE || e == Epi::TANH_GRAD) &&
        (N & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
        (!aux || (reinterpret_cast<uintptr_t>(aux) & 15) == 0)) {
        // rows per CTA: up to 32, but at least ~2 CTAs per SM
        const int colblocks = (N / 4 + 255) / 256;
        int rows = (M / std::max(1, (2 * g.sm_count + colblocks - 1) / colblocks)) & ~3;
        rows = std::max(4, std::min(kShortRows, rows));
        const dim3 grid(colblocks, (M + rows - 1) / rows);
        if (e == Epi::STORE)
            k_gemm_shortk_nt4<Epi::STORE><<<grid, 256, 0, g.stream>>>(M, N, K, A, B, C, nullptr, rows);
        else
            k_gemm_shortk_nt4<Epi::TANH_GRAD><<<grid, 256, 0, g.stream>>>(M, N, K, A, B, C, aux, rows);
        *g.launches += 1;
        return true;
    }
    if (op == GemmOp::NT && K <= kShortK && lda == K && ldb == K && (e == Epi::STORE || e == Epi::TANH_GRAD)) {
        const dim3 grid((N + 255) / 256, (M + 7) / 8);
        if (e == Epi::STORE)
            k_gemm_shortk_nt<Epi::STORE><<<grid, 256, 0, g.stream>>>(M, N, K, A, B, C, nullptr);
        else
            k_gemm_shortk_nt<Epi::TANH_GRAD><<<grid, 256, 0, g.stream>>>(M, N, K, A, B, C, aux);
        *g.launches += 1;
        return true;
    }
    if (N > 32) return false;
    if (op == GemmOp::NN && lda == K && ldb == N && e != Epi::TANH_GRAD && N <= 16 && K >= 2 * kSkKC &&
        M >= 2048 && K % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
        // enough rows for >= 8 row blocks x the K chunks (C3's 256 rows stay on
        // the lanes-along-K kernel below: 7 us there against 13 us here)
        const int S = (K + kSrKC - 1) / kSrKC;
        ensure_ws(g, (size_t)S * M * N);
        k_gemm_skinny_nn_rows<<<dim3((M + 255) / 256, S), 256, 0, g.stream>>>(M, N, K, A, B, *g.ws);
        const int blocks = std::max(1, std::min(4 * g.sm_count, (M * N + 255) / 256));
        switch (e) {
            case Epi::STORE: k_sum_partials_epi<Epi::STORE><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
            case Epi::BIAS: k_sum_partials_epi<Epi::BIAS><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
            default: k_sum_partials_epi<Epi::BIAS_TANH><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
        }
        *g.launches += 2;
        return true;
    }
    if (op == GemmOp::NN && lda == K && ldb == N && e != Epi::TANH_GRAD && N <= 16 && K >= 2 * kSkKC) {
        // long K: chunked, B chunk in shared memory, fixed-order partial sum
        const int S = (K + kSkKC - 1) / kSkKC;
        ensure_ws(g, (size_t)S * M * N);
        // one row per warp: several rows per warp (less B staging) measured
        // slower at C5's 4096 x 10 x 4096 (70.7 vs 65 us)
        const int rpw = 1;
        k_gemm_skinny_nn_kc<<<dim3((M + 8 * rpw - 1) / (8 * rpw), S), 256, 0, g.stream>>>(M, N, K, A, B, *g.ws, rpw);
        const int blocks = std::max(1, std::min(4 * g.sm_count, (M * N + 255) / 256));
        switch (e) {
            case Epi::STORE: k_sum_partials_epi<Epi::STORE><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
            case Epi::BIAS: k_sum_partials_epi<Epi::BIAS><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
            default: k_sum_partials_epi<Epi::BIAS_TANH><<<blocks, 256, 0, g.stream>>>(*g.ws, S, M, N, C, C2, bias); break;
        }
        *g.launches += 2;
        return true;
    }
    if (op == GemmOp::NN && lda == K && ldb == N && e != Epi::TANH_GRAD) {
        const int blocks = std::max(1, std::min(16 * g.sm_count, M));
        constexpr int T = 32 * kSkNW;
        switch (e) {
            case Epi::STORE: k_gemm_skinny_nn<Epi::STORE><<<blocks, T, 0, g.stream>>>(M, N, K, A, B, C, C2, bias); break;
            case Epi::BIAS: k_gemm_skinny_nn<Epi::BIAS><<<blocks, T, 0, g.stream>>>(M, N, K, A, B, C, C2, bias); break;
            default: k_gemm_skinny_nn<Epi::BIAS_TANH><<<blocks, T, 0, g.stream>>>(M, N, K, A, B, C, C2, bias); break;
        }
        *g.launches += 1;
        return true;
    }
    if (op == GemmOp::TN && lda == M && ldb == N && e == Epi::STORE && (M + 31) / 32 >= g.sm_count / 2 &&
        K <= 4 * kSkinnyKChunk) {
        // enough row blocks to fill the GPU: one pass over K, no partials
        const int S = (K + kSkinnyKChunk - 1) / kSkinnyKChunk;
        if (N <= 16)
            k_gemm_skinny_tn<16><<<dim3((M + 31) / 32, 1), 32 * skinny_tn_warps<16>(), 0, g.stream>>>(M, N, K, A, B, C, S);
        else
            k_gemm_skinny_tn<32><<<dim3((M + 31) / 32, 1), 32 * kSkTnW, 0, g.stream>>>(M, N, K, A, B, C, S);
        *g.launches += 1;
        return true;
    }
    if (op == GemmOp::TN && lda == M && ldb == N && e == Epi::STORE) {
        const int S = (K + kSkinnyKChunk - 1) / kSkinnyKChunk;
        ensure_ws(g, (size_t)S * M * N);
        if (N <= 16)
            k_gemm_skinny_tn<16><<<dim3((M + 31) / 32, S), 32 * skinny_tn_warps<16>(), 0, g.stream>>>(M, N, K, A, B,
                                                                                                   *g.ws, 1);
        else
            k_gemm_skinny_tn<32><<<dim3((M + 31) / 32, S), 32 * kSkTnW, 0, g.stream>>>(M, N, K, A, B, *g.ws, 1);
        k_sum_partials<<<std::max(1, std::min(4 * g.sm_count, (M * N + 255) / 256)), 256, 0, g.stream>>>(
            *g.ws, S, (size_t)M * N, C);
        *g.launches += 2;
        return true;
    }
    return false;
}

// 0 = SIMT only, 1 = tensor cores where eligible (default), set by
// LANE_B200_GEMM=simt|tc or lane_b200_gemm()'s use_tc argument
inline int& gemm_tc_mode() {
    static int mode = [] {
        const char* e = std::getenv("LANE_B200_GEMM");
        return (e && std::strcmp(e, "simt") == 0) ? 0 : 1;
    }();
    return mode;
}

// 1 = the persistent stream-K kernel (gemm_tcp.cuh) serves the single-CTA
// shapes and the short-K wgrads (default); 0 = never; 2 = every shape
// (lane_b200_gemm's use_tc = 2 / 3 select 2 / 0 for one call)
inline int& tc_persist_mode() {
    static int persist = std::getenv("LANE_B200_TC_PERSIST") ? std::atoi(std::getenv("LANE_B200_TC_PERSIST")) : 1;
    return persist;
}

// CTA pairs (cta_group::2, 256 x 256 tiles, N = 256 MMAs) for the tall
// GEMMs: 4096^3 0.596 -> 0.500 ms.  The M = 256 GEMMs stay on single CTAs (a
// 256-row pair tile leaves 16 tiles for 148 SMs), and the short-K wgrads
// (K = batch <= 1024) run on the persistent kernel, whose double-buffered
// accumulators overlap each tile's epilogue with the next tile's MMAs and
// whose epilogue can carry the fused SGD/momentum update.
inline bool tc_use_pair(GemmOp op, int M, int N, int K) {
    static const bool pair_ok = !std::getenv("LANE_B200_TC_NOPAIR");
    const int persist = tc_persist_mode();
    if (!pair_ok || persist == 2) return false;
    if (persist == 1 && op == GemmOp::TN && K <= 1024) return false;
    static const int min_m = std::getenv("LANE_B200_TC_PAIR_MIN_M") ? std::atoi(std::getenv("LANE_B200_TC_PAIR_MIN_M")) : 0;
    if (min_m > 0) return M >= min_m;
    return M >= 1024 || (M >= 512 && K >= 2048);
}

// Tensor-core operand precision scheme: 0 = 3xTF32 everywhere (gemm_tc.cuh /
// gemm_tcp.cuh); 1 = 3xF16 with power-of-two row/column scales (gemm_h3.cuh)
// everywhere; 2 (default) = 3xF16 for the tall CTA-pair shapes with a long K
// (4096^3: 0.51 -> 0.38 ms including the operand-maxima passes), 3xTF32 for
// the rest (the M = batch = 256 shapes and short-K wgrads of C3 run faster on
// the persistent stream-K 3xTF32 kernel).  LANE_B200_TC_PREC=tf32|f16|auto,
// or lane_b200_gemm()'s use_tc = 4 (3xF16) for one call.
inline int& tc_prec_mode() {
    static int mode = [] {
        const char* e = std::getenv("LANE_B200_TC_PREC");
        if (e && std::strcmp(e, "f16") == 0) return 1;
        if (e && std::strcmp(e, "tf32") == 0) return 0;
        return 2;
    }();
    return mode;
}
inline bool tc_use_h3(int M, int N, int K) {
    const int m = tc_prec_mode();
    static const int min_m = std::getenv("LANE_B200_H3_MIN_M") ? std::atoi(std::getenv("LANE_B200_H3_MIN_M")) : 0;
    if (m == 2 && min_m > 0) return M >= min_m && K >= 2048 && N >= 256;
    return m == 1 || (m == 2 && (M >= 1024 || (M >= 512 && K >= 2048)) && K >= 2048 && N >= 256);
}

// 3xF16: per-row maxima of op(A) and per-column maxima of op(B) into the
// workspace tail, then the split-scaled kernel (pairs for the tall shapes,
// single CTAs with split-K otherwise)
inline void gemm_h3(GemmCtx& g, GemmOp op, int M, int N, int K, const float* A, const float* B, Epi e, float* C,
                    float* C2, const float* bias, const float* aux, const GemmMax* mx, bool* fused_out) {
    static const int pair_min_m = std::getenv("LANE_B200_H3_PAIR_MIN_M") ? std::atoi(std::getenv("LANE_B200_H3_PAIR_MIN_M")) : 0;
    const bool pair = pair_min_m > 0 ? M >= pair_min_m : (M >= 1024 || (M >= 512 && K >= 2048));
    CUtensorMap ma, mb;
    bool a_mn = false, b_mn = false;
    switch (op) {
        case GemmOp::NN:
            ma = tc_map(A, M, K, 32, 128, 0);
            mb = tc_map(B, K, N, 128, 32, 2);
            b_mn = true;
            break;
        case GemmOp::NT:
            ma = tc_map(A, M, K, 32, 128, 0);
            mb = tc_map(B, N, K, 32, 128, 0);
            break;
        case GemmOp::TN:
            ma = tc_map(A, K, M, 128, 32, 2);
            mb = tc_map(B, K, N, 128, 32, 2);
            a_mn = b_mn = true;
            break;
    }
    TcArgs t{M, N, K, 0, nullptr, C, C2, bias, aux};
    constexpr int kPN = H3Cfg<true>::kBN;
    const int tiles = pair ? 2 * ((M + 2 * kTcBM - 1) / (2 * kTcBM)) * ((N + kPN - 1) / kPN)
                           : ((M + kTcBM - 1) / kTcBM) * ((N + kTcBN - 1) / kTcBN);
    const int nkb = (K + kTcBK - 1) / kTcBK;
    static const int kbmin = std::getenv("LANE_B200_TC_SPLITK_KBMIN") ? std::atoi(std::getenv("LANE_B200_TC_SPLITK_KBMIN")) : 24;
    static const int h3_smax = std::getenv("LANE_B200_H3_SPLITK_MAX") ? std::atoi(std::getenv("LANE_B200_H3_SPLITK_MAX")) : 4;
    int S = std::max(1, std::min({h3_smax, g.sm_count / std::max(1, tiles), nkb / kbmin}));
    if (K % kTcBK != 0) S = 1;
    size_t part = 0;
    if (S > 1) {
        t.kbs = (nkb + S - 1) / S;
        S = (nkb + t.kbs - 1) / t.kbs;
        part = (size_t)S * M * N;
    }
    // tail-wave split (pairs, no split-K): when the last wave of pair tiles is
    // at most half full, its tiles run as two K halves each (twice as many
    // units, half as long), then k_h3_tail_reduce sums the halves in a fixed
    // order and applies the epilogue.  C5's 4096^3: 256 tiles on 74 pairs =
    // 3 full waves + 34 tiles -> 3.5 wave-times instead of 4.
    static const bool tail_ok = std::getenv("LANE_B200_H3_NOTAIL") == nullptr;
    size_t tail_floats = 0;
    if (pair && S == 1 && tail_ok && nkb >= 16) {
        const int tm = (M + 2 * kTcBM - 1) / (2 * kTcBM), tn = (N + kPN - 1) / kPN;
        const int T = tm * tn, P = std::max(1, g.sm_count / 2);
        const int full = (T / P) * P, tail = T - full;
        if (full > 0 && tail > 0 && 2 * tail <= P) {
            t.full_units = full;
            t.tiles_m = tm;
            t.tiles_n = tn;
            tail_floats = (size_t)tail * 2 * 65536;
        }
    }
    // [split-K partials or tail-wave halves | row maxima of op(A) | column maxima of op(B)]
    part = std::max(part, tail_floats);
    ensure_ws(g, part + (size_t)M + (size_t)N);
    float* ws = *g.ws;
    if (S > 1) t.part = ws;
    if (t.full_units > 0) {
        t.tail_part = ws;
        *g.launches += 1;  // the tail reduce
    }
    unsigned* amax = reinterpret_cast<unsigned*>(ws + part);
    unsigned* bmax = amax + M;
    if (mx && mx->a) {
        t.amax = mx->a;
    } else {
        absmax_launch(g.stream, A, op == GemmOp::TN ? K : M, op == GemmOp::TN ? M : K, op != GemmOp::TN, amax);
        t.amax = amax;
        *g.launches += 1;
    }
    if (mx && mx->b) {
        t.bmax = mx->b;
    } else {
        absmax_launch(g.stream, B, op == GemmOp::NT ? N : K, op == GemmOp::NT ? K : N, op == GemmOp::NT, bmax);
        t.bmax = bmax;
        *g.launches += 1;
    }
    if (mx && mx->orow && S == 1) {  // the tail reduce emits its tiles' maxima too
        t.omax_row = mx->orow;
        t.omax_col = mx->ocol;
        *fused_out = true;
    }
    static const int diag = std::getenv("LANE_B200_H3_DIAG") ? std::atoi(std::getenv("LANE_B200_H3_DIAG")) : 0;
    t.diag = diag;
    if (mx && e == Epi::STORE) t.out_scale = mx->out_scale;
    *g.launches += S > 1 ? 1 : 0;
    // the epilogue's TMA store boxes: 32 columns x 32 rows, 128-byte swizzle
    const CUtensorMap mc = tc_map(C, M, N, 32, 32, 0);
    // C2: tanh(z) for the forward; for the dgrad, the activations its
    // epilogue reads (TMA-prefetched into the landing ring, 32 x 32 boxes)
    const CUtensorMap mc2 = e == Epi::BIAS_TANH   ? tc_map(C2, M, N, 32, 32, 0)
                            : e == Epi::TANH_GRAD ? tc_map(aux, M, N, 32, 32, 0)
                                                  : mc;
    switch (e) {
        case Epi::STORE:
            if (pair) h3_dispatch<TcEpi::STORE, true>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            else h3_dispatch<TcEpi::STORE, false>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            break;
        case Epi::BIAS:
            if (pair) h3_dispatch<TcEpi::BIAS, true>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            else h3_dispatch<TcEpi::BIAS, false>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            break;
        case Epi::BIAS_TANH:
            if (pair) h3_dispatch<TcEpi::BIAS_TANH, true>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            else h3_dispatch<TcEpi::BIAS_TANH, false>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            break;
        case Epi::TANH_GRAD:
            if (pair) h3_dispatch<TcEpi::TANH_GRAD, true>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            else h3_dispatch<TcEpi::TANH_GRAD, false>(g.stream, a_mn, b_mn, ma, mb, mc, mc2, t);
            break;
    }
    *g.launches += 1;
}

// Whether gemm() runs this call on the 3xF16 kernel (the step uses it to
// decide which operand maxima to provide).
inline bool gemm_will_h3(GemmOp op, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                         const float* C) {
    if (!gemm_tc_mode() || !tc_eligible(M, N, K) || !tc_use_h3(M, N, K)) return false;
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
        return false;
    return lda == (op == GemmOp::TN ? M : K) && ldb == (op == GemmOp::NT ? K : N);
}

// Tensor-core dispatch (gemm_tc.cuh): returns false when the shape/layout is
// not eligible (the caller then runs the SIMT kernel).
inline bool gemm_try_tc(GemmCtx& g, GemmOp op, int M, int N, int K, const float* A, int lda, const float* B,
                        int ldb, Epi e, float* C, float* C2, const float* bias, const float* aux,
                        const GemmMax* mx = nullptr, bool* fused = nullptr) {
    if (!gemm_tc_mode() || !tc_eligible(M, N, K)) return false;
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C) |
         reinterpret_cast<uintptr_t>(C2) | reinterpret_cast<uintptr_t>(aux)) & 15)
        return false;
    if (gemm_will_h3(op, M, N, K, A, lda, B, ldb, C)) {
        bool f = false;
        gemm_h3(g, op, M, N, K, A, B, e, C, C2, bias, aux, mx, &f);
        if (fused) *fused = f;
        return true;
    }
    CUtensorMap ma, mb;
    bool a_mn = false, b_mn = false;
    const bool pair = tc_use_pair(op, M, N, K);
    switch (op) {
        case GemmOp::NN:  // A [M][K] K-major, B [K][N] MN-major
            if (lda != K || ldb != N) return false;
            ma = tc_map(A, M, K, 32, 128, 0);
            mb = tc_map(B, K, N, 32, 32, 1);
            b_mn = true;
            break;
        case GemmOp::NT:  // A [M][K] K-major, B [N][K] K-major
            if (lda != K || ldb != K) return false;
            ma = tc_map(A, M, K, 32, 128, 0);
            mb = tc_map(B, N, K, 32, TcCfg<false>::kBN, 0);  // 128 rows: a pair CTA's half of a 256 tile
            break;
        case GemmOp::TN:  // A [K][M] MN-major, B [K][N] MN-major
            if (lda != M || ldb != N) return false;
            ma = tc_map(A, K, M, 128, 32, 2);
            mb = tc_map(B, K, N, 32, 32, 1);
            a_mn = b_mn = true;
            break;
    }
    // the persistent kernel (gemm_tcp.cuh) for the short-K wgrads (mode 1) or
    // every shape (mode 2); the M = batch forward/dgrad GEMMs stay on the
    // one-tile-per-CTA kernel with split-K, measured faster there (C3
    // 256x4096x4096: 60.5 vs 65.6 us; 256x4096x1024: 25.5 vs 37.8 us)
    if (tc_persist_mode() == 2 || (tc_persist_mode() == 1 && op == GemmOp::TN && K <= 1024 && !pair)) {
        TpPlan p = tp_plan(M, N, K, g.sm_count);
        bool ok = true;
        if (p.a.sk) {
            ok = ensure_counters(g, (size_t)p.tiles);
            if (ok) {
                ensure_ws(g, p.part_floats);
                p.a.part = *g.ws;
                p.a.counters = *g.counters;
            }
        }
        if (ok) {
            p.a.C = C;
            p.a.C2 = C2;
            p.a.bias = bias;
            p.a.aux = aux;
            switch (e) {
                case Epi::STORE: tp_dispatch<TpEpi::STORE>(g.stream, a_mn, b_mn, ma, mb, p); break;
                case Epi::BIAS: tp_dispatch<TpEpi::BIAS>(g.stream, a_mn, b_mn, ma, mb, p); break;
                case Epi::BIAS_TANH: tp_dispatch<TpEpi::BIAS_TANH>(g.stream, a_mn, b_mn, ma, mb, p); break;
                case Epi::TANH_GRAD: tp_dispatch<TpEpi::TANH_GRAD>(g.stream, a_mn, b_mn, ma, mb, p); break;
            }
            *g.launches += 1;
            return true;
        }
    }
    TcArgs t{M, N, K, 0, nullptr, C, C2, bias, aux};
    // split-K when the 128x128 tiles fill less than half the SMs (the M = batch
    // GEMMs at B = 256): S splits of >= 24 K blocks each, <= 4, one wave
    // CTAs per split: pairs run 256 x 256 tiles on 2 CTAs
    constexpr int kPN = TcCfg<true>::kBN;
    const int tiles = pair ? 2 * ((M + 2 * kTcBM - 1) / (2 * kTcBM)) * ((N + kPN - 1) / kPN)
                           : ((M + kTcBM - 1) / kTcBM) * ((N + kTcBN - 1) / kTcBN);
    const int nkb = K / kTcBK;
    static const int smax = std::getenv("LANE_B200_TC_SPLITK_MAX") ? std::atoi(std::getenv("LANE_B200_TC_SPLITK_MAX")) : 4;
    // split while every split keeps >= 8 K blocks: with float4 partial stores
    // C3 runs 836k samples/s at a 24-block minimum, 857k at 8 (its
    // 256x4096x1024 forward splits in 4; with scalar partial stores the
    // unsplit forward had been faster)
    static const int kbmin = std::getenv("LANE_B200_TC_SPLITK_KBMIN") ? std::atoi(std::getenv("LANE_B200_TC_SPLITK_KBMIN")) : 8;
    int S = std::min({smax, g.sm_count / std::max(1, tiles), nkb / kbmin});
    if (K % kTcBK != 0 || (N & 3) != 0) S = 1;
    if (S > 1) {
        t.kbs = (nkb + S - 1) / S;
        S = (nkb + t.kbs - 1) / t.kbs;
        ensure_ws(g, (size_t)S * M * N);
        t.part = *g.ws;
        *g.launches += 1;  // the split-K reduce
    }
    switch (e) {
        case Epi::STORE:
            if (pair) tc_dispatch<TcEpi::STORE, true>(g.stream, a_mn, b_mn, ma, mb, t);
            else tc_dispatch<TcEpi::STORE, false>(g.stream, a_mn, b_mn, ma, mb, t);
            break;
        case Epi::BIAS:
            if (pair) tc_dispatch<TcEpi::BIAS, true>(g.stream, a_mn, b_mn, ma, mb, t);
            else tc_dispatch<TcEpi::BIAS, false>(g.stream, a_mn, b_mn, ma, mb, t);
            break;
        case Epi::BIAS_TANH:
            if (pair) tc_dispatch<TcEpi::BIAS_TANH, true>(g.stream, a_mn, b_mn, ma, mb, t);
            else tc_dispatch<TcEpi::BIAS_TANH, false>(g.stream, a_mn, b_mn, ma, mb, t);
            break;
        case Epi::TANH_GRAD:
            if (pair) tc_dispatch<TcEpi::TANH_GRAD, true>(g.stream, a_mn, b_mn, ma, mb, t);
            else tc_dispatch<TcEpi::TANH_GRAD, false>(g.stream, a_mn, b_mn, ma, mb, t);
            break;
    }
    *g.launches += 1;
    return true;
}

// wgrad fused with the SGD/momentum update (TN: G[M,N] = A[K,M]^T B[K,N] / B_glob,
// then V = mu V - eta G, W += V), on the persistent tensor-core kernel only.
// Returns false (nothing launched) when the shape or layout is not eligible.
inline bool gemm_wgrad_update(GemmCtx& g, int M, int N, int K, const float* A, const float* B, float* G, float* W,
                              float* V, float inv_b, float neg_eta, float mu) {
    static const bool fuse = !std::getenv("LANE_B200_NO_FUSED_UPDATE");
    if (!fuse || !tc_persist_mode() || !gemm_tc_mode() || tc_use_h3(M, N, K) || !tc_eligible(M, N, K)) return false;
    if (tc_use_pair(GemmOp::TN, M, N, K)) return false;  // the wgrad stays on the pair kernel
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(G) |
         reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(V)) & 15)
        return false;
    TpPlan p = tp_plan(M, N, K, g.sm_count);
    if (p.a.sk) {
        if (!ensure_counters(g, (size_t)p.tiles)) return false;
        ensure_ws(g, p.part_floats);
        p.a.part = *g.ws;
        p.a.counters = *g.counters;
    }
    const CUtensorMap ma = tc_map(A, K, M, 128, 32, 2);
    const CUtensorMap mb = tc_map(B, K, N, 32, 32, 1);
    p.a.C = G;
    p.a.W = W;
    p.a.V = V;
    p.a.inv_b = inv_b;
    p.a.neg_eta = neg_eta;
    p.a.mu = mu;
    tp_dispatch<TpEpi::UPDATE>(g.stream, true, true, ma, mb, p);
    *g.launches += 1;
    return true;
}

inline void gemm(GemmCtx& g, GemmOp op, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                 Epi e, float* C, float* C2, const float* bias, const float* aux, const GemmMax* mx = nullptr) {
    if (M <= 0 || N <= 0) return;
    bool fused = false;
    if (mx && mx->out_scale != 0.0f && (e != Epi::STORE || !gemm_will_h3(op, M, N, K, A, lda, B, ldb, C)))
        throw Error(LANE_ERR_CONFIG, "gemm: out_scale is a 3xF16 STORE option");
    if (gemm_try_tc(g, op, M, N, K, A, lda, B, ldb, e, C, C2, bias, aux, mx, &fused)) {
    } else if (gemm_try_skinny(g, op, M, N, K, A, lda, B, ldb, e, C, C2, bias, aux)) {
    } else {
        switch (op) {
            case GemmOp::NN: gemm_simt_dispatch<GemmOp::NN>(g, M, N, K, A, lda, B, ldb, e, C, C2, bias, aux); break;
            case GemmOp::NT: gemm_simt_dispatch<GemmOp::NT>(g, M, N, K, A, lda, B, ldb, e, C, C2, bias, aux); break;
            case GemmOp::TN: gemm_simt_dispatch<GemmOp::TN>(g, M, N, K, A, lda, B, ldb, e, C, C2, bias, aux); break;
        }
    }
    if (mx && mx->orow && !fused) {
        // the output's maxima in one extra pass (zeroed by the caller)
        absmax_rc_launch(g.stream, e == Epi::BIAS_TANH ? C2 : C, M, N, mx->orow, mx->ocol);
        *g.launches += 1;
    }
}

}  // namespace lane_b200
