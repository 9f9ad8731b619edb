// Latency micro-benchmarks for the online-SGD critical chain (one warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_chain.cu && /tmp/ubench
// Each test runs a dependent chain of N steps in one warp and prints cycles/step.
#include <cstdio>
#include <cuda_runtime.h>

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
    return 0;
}
