// Latency micro-benchmarks for the online-SGD critical chain (one warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_chain.cu && /tmp/ubench
// Each test runs a dependent chain of N steps in one warp and prints cycles/step.
#include <cstdio>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

constexpr int N = 4096;

__device__ __forceinline__ float tanh_poly_exp(float x) {
    const float ax = fabsf(x);
    const float u = x * x;
    float p = -0.00035334646f;
    p = fmaf(p, u, 0.0022822332f);
    p = fmaf(p, u, -0.0079174498f);
    p = fmaf(p, u, 0.021464825f);
    p = fmaf(p, u, -0.053870916f);
    p = fmaf(p, u, 0.13332160f);
    p = fmaf(p, u, -0.33333278f);
    const float small = fmaf(x * u, p, x);
    float t;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(ax * -2.8853900817779268f));
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + t));
    const float big = copysignf((1.0f - t) * r, x);
    return ax < 1.0f ? small : big;
}

__device__ __forceinline__ float tanh_rational(float x) {
    x = fminf(fmaxf(x, -7.90531110763549805f), 7.90531110763549805f);
    const float x2 = x * x;
    float p = -2.76076847742355e-16f;
    p = fmaf(x2, p, 2.00018790482477e-13f);
    p = fmaf(x2, p, -8.60467152213735e-11f);
    p = fmaf(x2, p, 5.12229709037114e-08f);
    p = fmaf(x2, p, 1.48572235717979e-05f);
    p = fmaf(x2, p, 6.37261928875436e-04f);
    p = fmaf(x2, p, 4.89352455891786e-03f);
    p = x * p;
    float q = fmaf(x2, 1.19825839466702e-06f, 1.18534705686654e-04f);
    q = fmaf(x2, q, 2.26843463243900e-03f);
    q = fmaf(x2, q, 4.89352518554385e-03f);
    return __fdividef(p, q);
}

__device__ __forceinline__ float tanh_approx(float x) {
    float r;
    asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int T>
__global__ void k_bench(float* out, long long* cyc, float seed) {
    const int lane = threadIdx.x;
    float v0 = seed * (lane + 1) * 0.01f, v1 = v0 + 0.1f, v2 = v0 - 0.2f, v3 = v0 + 0.3f;
    __shared__ float sh[64];
    sh[lane] = v0;
    sh[lane + 32] = v1;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        if constexpr (T == 0) {  // CUDA tanhf x4 (independent)
            v0 = tanhf(v0 * 1.7f); v1 = tanhf(v1 * 1.7f); v2 = tanhf(v2 * 1.7f); v3 = tanhf(v3 * 1.7f);
        } else if constexpr (T == 1) {
            v0 = tanh_poly_exp(v0 * 1.7f); v1 = tanh_poly_exp(v1 * 1.7f);
            v2 = tanh_poly_exp(v2 * 1.7f); v3 = tanh_poly_exp(v3 * 1.7f);
        } else if constexpr (T == 2) {
            v0 = tanh_rational(v0 * 1.7f); v1 = tanh_rational(v1 * 1.7f);
            v2 = tanh_rational(v2 * 1.7f); v3 = tanh_rational(v3 * 1.7f);
        } else if constexpr (T == 3) {
            v0 = tanh_approx(v0 * 1.7f); v1 = tanh_approx(v1 * 1.7f);
            v2 = tanh_approx(v2 * 1.7f); v3 = tanh_approx(v3 * 1.7f);
        } else if constexpr (T == 4) {  // one shfl_xor round (dependent)
            v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
        } else if constexpr (T == 5) {  // expf
            v0 = expf(v0 * -0.5f);
        } else if constexpr (T == 6) {  // __fdiv_rn
            v0 = __fdiv_rn(1.0f, v0 + 1.5f);
        } else if constexpr (T == 7) {  // __frcp_rn
            v0 = __frcp_rn(v0 + 1.5f);
        } else if constexpr (T == 8) {  // smem load (dependent)
            v0 = sh[(__float_as_uint(v0) & 31)] + 1e-30f;
        } else if constexpr (T == 9) {  // fma chain
            v0 = fmaf(v0, 0.999f, 0.001f);
        } else if constexpr (T == 10) {  // redux.sync.max.f32? use u32 add redux
            unsigned r;
            asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(__float_as_uint(v0)));
            v0 = __uint_as_float((r & 0x3fffffffu) | 0x3f800000u);
        } else if constexpr (T == 11) {  // __expf
            v0 = __expf(v0 * -0.5f);
        } else if constexpr (T == 12) {  // __fdividef
            v0 = __fdividef(1.0f, v0 + 1.5f);
        }
    }
    long long t1 = clock64();
    out[lane] = v0 + v1 + v2 + v3;
    if (lane == 0) cyc[T] = t1 - t0;
}

// The C2 sample chain's critical path only (784-128-10: one warp, 4 hidden
// units per lane, 10 classes), with none of the off-chain work the window
// kernel's chain warp also issues (the deferred W1 update, the fetch of the
// next row, the bias / statistics bookkeeping):
//   z = c1 d0(s-1) + y + b0; a = tanh z; partial logits (4 FMA x 10) ->
//   transposed smem tile -> lane k sums class k (8 LDS.128 + tree) -> + b1 ->
//   redux max -> exp -> smem -> every lane sums the 10 exponentials -> rcp ->
//   d1 = p - t -> d0 = (1 - a^2) (W1 d1) -> next z.
// cycles/step of this kernel is the dependency floor a one-warp chain of this
// algorithm cannot beat (bench.py's C2 line reports it as roofline.latency).
__global__ void k_chain_floor(float* out, long long* cyc, float seed, int n) {
    constexpr int C = 10, CC = 10, XS = 36;
    __shared__ __align__(16) float xr[16 * XS];
    __shared__ __align__(16) float es[16];
    const int lane = threadIdx.x;
    const bool kval = lane < C;
    const int kr = lane & 15;
    float w1[4][CC], y[4], b0r[4], dp1[4], t[CC];
    for (int m = 0; m < 4; ++m) {
        for (int k = 0; k < CC; ++k) w1[m][k] = seed * 0.01f * (float)((lane * 4 + m) * 7 + k * 3 - 40) / 64.0f;
        y[m] = seed * 0.1f * (lane - 16) / 16.0f;
        b0r[m] = 0.01f * m;
        dp1[m] = 0.0f;
    }
    for (int k = 0; k < CC; ++k) t[k] = k == 3 ? 1.0f : 0.0f;
    for (int e = lane; e < 16 * XS; e += 32) xr[e] = 0.0f;
    if (lane < 16) es[lane] = 0.0f;
    const float c1 = -0.01f * seed, b1k = 0.0f;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        float a[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) a[m] = tanhf(fmaf(c1, dp1[m], y[m]) + b0r[m]);
#pragma unroll
        for (int k = 0; k < CC; ++k) {
            float acc = 0.0f;
#pragma unroll
            for (int m = 0; m < 4; ++m) acc = fmaf(a[m], w1[m][k], acc);
            xr[k * XS + lane] = acc;
        }
        __syncwarp();
        const float4* col = reinterpret_cast<const float4*>(xr + kr * XS);
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = col[q];
        float t8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t8[q] = (v[q].x + v[q].y) + (v[q].z + v[q].w);
        const float zown = (((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]))) + b1k;
        float mx;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;\n" : "=f"(mx) : "f"(kval ? zown : -INFINITY));
        const float eown = expf(zown - mx);
        if (kval) es[lane] = eown;
        __syncwarp();
        float ek[12];
#pragma unroll
        for (int k4 = 0; k4 < 3; ++k4) {
            const float4 q = reinterpret_cast<const float4*>(es)[k4];
            ek[4 * k4] = q.x; ek[4 * k4 + 1] = q.y; ek[4 * k4 + 2] = q.z; ek[4 * k4 + 3] = q.w;
        }
        ek[10] = ek[11] = 0.0f;
        float sp[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) sp[k] = ek[k];
#pragma unroll
        for (int w = 1; w < 12; w <<= 1)
#pragma unroll
            for (int k = 0; k + w < 12; k += 2 * w) sp[k] += sp[k + w];
        float inv;
        asm volatile("rcp.approx.ftz.f32 %0, %1;\n" : "=f"(inv) : "f"(sp[0]));
        float d1[CC];
#pragma unroll
        for (int k = 0; k < CC; ++k) d1[k] = fmaf(ek[k], inv, -t[k]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
            for (int k = 0; k < CC / 2; ++k) acc0 = fmaf(d1[k], w1[m][k], acc0);
#pragma unroll
            for (int k = CC / 2; k < CC; ++k) acc1 = fmaf(d1[k], w1[m][k], acc1);
            dp1[m] = fmaf(-a[m], a[m], 1.0f) * (acc0 + acc1);
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[lane] = dp1[0] + dp1[1] + dp1[2] + dp1[3];
    if (lane == 0) cyc[15] = t1 - t0;
}

// The same critical path for the wide window plans (C4, H = NCW x CS x 128):
// NCW chain warps per CTA (each 128 hidden units, 4 per lane) and CS chain
// CTAs in one thread-block cluster.  Per sample, on top of the one-warp chain:
//   NCW > 1: per-warp class half sums -> shared memory, one named barrier,
//            every warp sums the NCW halves;
//   CS > 1:  chain warp 0 pushes the C slice partials to every peer with
//            st.async (completing the peer's exchange mbarrier), every warp
//            waits for all CS and sums them in rank order; the pusher re-arms
//            the barrier for sample s + 2 -- the window kernel's exchange.
template <int NCW, int CS>
__global__ void k_chain_floor_cl(float* out, long long* cyc, float seed, int n) {
    constexpr int C = 10, CC = 10, XS = 32 * NCW + 4, CP = 16;
    __shared__ __align__(16) float xr[16 * XS];
    __shared__ __align__(16) float half[2][NCW][CP];
    __shared__ __align__(16) float es[NCW][16];
    __shared__ __align__(16) float gat[2][16][CP];
    __shared__ __align__(8) unsigned long long xbar[2];
    const int lane = threadIdx.x & 31, cw = threadIdx.x >> 5;
    unsigned rank = 0;
    if (CS > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
    const bool kval = lane < C;
    const int kr = lane & 15;
    float w1[4][CC], y[4], b0r[4], dp1[4], t[CC];
    for (int m = 0; m < 4; ++m) {
        for (int k = 0; k < CC; ++k)
            w1[m][k] = seed * 0.01f * (float)(((cw * 32 + lane) * 4 + m) * 7 + k * 3 - 40) / 64.0f;
        y[m] = seed * 0.1f * (lane - 16) / 16.0f;
        b0r[m] = 0.01f * m;
        dp1[m] = 0.0f;
    }
    for (int k = 0; k < CC; ++k) t[k] = k == 3 ? 1.0f : 0.0f;
    for (int e = threadIdx.x; e < 16 * XS; e += 32 * NCW) xr[e] = 0.0f;
    const uint32_t xb0 = (uint32_t)__cvta_generic_to_shared(&xbar[0]);
    if (threadIdx.x == 0) {
        for (int p = 0; p < 2; ++p) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xb0 + 8 * p));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int p = 0; p < 2 && p < n; ++p)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xb0 + 8 * p),
                         "r"(CS * C * 4));
    }
    if (CS > 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    else
        __syncthreads();
    const float c1 = -0.01f * seed, b1k = 0.0f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        float a[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) a[m] = tanhf(fmaf(c1, dp1[m], y[m]) + b0r[m]);
#pragma unroll
        for (int k = 0; k < CC; ++k) {
            float acc = 0.0f;
#pragma unroll
            for (int m = 0; m < 4; ++m) acc = fmaf(a[m], w1[m][k], acc);
            xr[k * XS + cw * 32 + lane] = acc;
        }
        __syncwarp();
        const float4* col = reinterpret_cast<const float4*>(xr + kr * XS + cw * 32);
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = col[q];
        float t8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t8[q] = (v[q].x + v[q].y) + (v[q].z + v[q].w);
        float hs = ((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]));
        if (NCW > 1) {
            if (kval) half[i & 1][cw][lane] = hs;
            asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NCW) : "memory");
            float hsum = half[i & 1][0][kr];
#pragma unroll
            for (int c = 1; c < NCW; ++c) hsum += half[i & 1][c][kr];
            hs = hsum;
        }
        if (CS > 1) {
            const int par = i & 1;
            const uint32_t slot = (uint32_t)__cvta_generic_to_shared(&gat[par][rank][lane]);
            const uint32_t xb = xb0 + 8 * par;
            if (cw == 0 && kval)
                for (int p = 0; p < CS; ++p) {
                    uint32_t ra, rb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(slot), "r"(p));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(xb), "r"(p));
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(
                                     ra),
                                 "r"(__float_as_uint(hs)), "r"(rb)
                                 : "memory");
                }
            asm volatile(
                "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra W_%=;\n}\n" ::"r"(xb),
                "r"((uint32_t)((i >> 1) & 1))
                : "memory");
            if (cw == 0 && lane == 0 && i + 2 < n)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xb), "r"(CS * C * 4));
            float tot = gat[par][0][kr];
#pragma unroll
            for (int p = 1; p < CS; ++p) tot += gat[par][p][kr];
            hs = tot;
        }
        const float zown = hs + b1k;
        float mx;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;\n" : "=f"(mx) : "f"(kval ? zown : -INFINITY));
        const float eown = expf(zown - mx);
        if (kval) es[cw][lane] = eown;
        __syncwarp();
        float ek[12];
#pragma unroll
        for (int k4 = 0; k4 < 3; ++k4) {
            const float4 q = reinterpret_cast<const float4*>(es[cw])[k4];
            ek[4 * k4] = q.x; ek[4 * k4 + 1] = q.y; ek[4 * k4 + 2] = q.z; ek[4 * k4 + 3] = q.w;
        }
        ek[10] = ek[11] = 0.0f;
        float sp[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) sp[k] = ek[k];
#pragma unroll
        for (int w = 1; w < 12; w <<= 1)
#pragma unroll
            for (int k = 0; k + w < 12; k += 2 * w) sp[k] += sp[k + w];
        float inv;
        asm volatile("rcp.approx.ftz.f32 %0, %1;\n" : "=f"(inv) : "f"(sp[0]));
        float d1[CC];
#pragma unroll
        for (int k = 0; k < CC; ++k) d1[k] = fmaf(ek[k], inv, -t[k]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
            for (int k = 0; k < CC / 2; ++k) acc0 = fmaf(d1[k], w1[m][k], acc0);
#pragma unroll
            for (int k = CC / 2; k < CC; ++k) acc1 = fmaf(d1[k], w1[m][k], acc1);
            dp1[m] = fmaf(-a[m], a[m], 1.0f) * (acc0 + acc1);
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = dp1[0] + dp1[1] + dp1[2] + dp1[3];
    if (threadIdx.x == 0 && rank == 0) cyc[0] = t1 - t0;
    if (CS > 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int NCW, int CS>
double run_cl(float* out, long long* cyc) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(32 * NCW);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (CS > 8) cudaFuncSetAttribute(k_chain_floor_cl<NCW, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_chain_floor_cl<NCW, CS>, out, cyc, 0.3f, N);
        if (e != cudaSuccess) {
            printf("launch NCW=%d CS=%d: %s\n", NCW, CS, cudaGetErrorString(e));
            return -1;
        }
        cudaDeviceSynchronize();
        best = std::min(best, (double)cyc[0] / N);
    }
    return best;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 32 * sizeof(float));
    cudaMallocManaged(&cyc, 16 * sizeof(long long));
    const char* names[] = {"tanhf x4", "poly|exp tanh x4", "rational tanh x4", "tanh.approx x4",
                           "shfl_xor round", "expf", "__fdiv_rn", "__frcp_rn", "LDS dep", "FFMA dep",
                           "redux.add.u32", "__expf", "__fdividef"};
    for (int rep = 0; rep < 2; ++rep) {
        k_bench<0><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<1><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<2><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<3><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<4><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<5><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<6><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<7><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<8><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<9><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<10><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<11><<<1, 32>>>(out, cyc, 0.3f);
        k_bench<12><<<1, 32>>>(out, cyc, 0.3f);
        cudaDeviceSynchronize();
    }
    for (int t = 0; t < 13; ++t) printf("%-20s %7.1f cycles/step\n", names[t], (double)cyc[t] / N);
    for (int rep = 0; rep < 3; ++rep) {
        k_chain_floor<<<1, 32>>>(out, cyc, 0.3f, N);
        cudaDeviceSynchronize();
    }
    printf("%-20s %7.1f cycles/step\n", "c2 chain floor", (double)cyc[15] / N);
    const double c2 = (double)cyc[15] / N;
    // the wide window plans of C4 (340-H-10): H -> (chain warps per CTA, cluster CTAs)
    const double h256 = run_cl<2, 1>(out, cyc), h512 = run_cl<1, 4>(out, cyc), h1024 = run_cl<1, 8>(out, cyc);
    const double h2048 = run_cl<1, 16>(out, cyc), h4096 = run_cl<2, 16>(out, cyc), h8192 = run_cl<4, 16>(out, cyc);
    printf("c4 floors: 256 %.1f 512 %.1f 1024 %.1f 2048 %.1f 4096 %.1f 8192 %.1f cycles/sample\n", h256, h512, h1024,
           h2048, h4096, h8192);
    printf("{\"c2_chain_floor_cycles\": %.1f, \"c4-256\": %.1f, \"c4-512\": %.1f, \"c4-1024\": %.1f, "
           "\"c4-2048\": %.1f, \"c4-4096\": %.1f, \"c4-8192\": %.1f}\n",
           c2, h256, h512, h1024, h2048, h4096, h8192);
    return 0;
}
