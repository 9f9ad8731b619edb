// common.cuh -- shared helpers for the lane_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/lane_b200.h"
#include "lane_libm.cuh"

namespace lane_b200 {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define LANE_CUDA(call)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::lane_b200::Error(LANE_ERR_CUDA, std::string(#call) + ": " +          \
                                                        cudaGetErrorString(e_));         \
    } while (0)

#define LANE_REQUIRE(cond, code, msg)                                                    \
    do {                                                                                 \
        if (!(cond)) throw ::lane_b200::Error((code), (msg));                            \
    } while (0)

constexpr int kWarp = 32;

// ---- reference-order arithmetic ------------------------------------------
// The reference objects are built without FMA: every a*b+c rounds
// twice.  These intrinsics are never contracted by nvcc, so STRICT kernels
// reproduce the reference bit-for-bit whatever -fmad says.
__device__ __forceinline__ float smul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float ssub(float a, float b) { return __fsub_rn(a, b); }

// -eta * (delta * x), then w + that: layers.hpp:34-35 / :55-56 and
// layers.cpp:20 -- three separately rounded operations.
__device__ __forceinline__ float sgd_apply(float w, float neg_eta, float delta, float x) {
    return sadd(w, smul(neg_eta, smul(delta, x)));
}

// (1 - a*a) * s  (layers.hpp:53)
__device__ __forceinline__ float tanh_grad(float a, float s) {
    return smul(ssub(1.0f, smul(a, a)), s);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// std::max(a, b) == (a < b) ? b : a  (NaN-propagation identical to the reference)
__device__ __forceinline__ float ref_max(float a, float b) { return (a < b) ? b : a; }

}  // namespace lane_b200
