// Batch input pipeline of the mini-batch trainer.
//
// kSlots page-locked host buffers and kSlots device buffers, one copy stream.
// For step s (slot s % kSlots) the host thread gathers the step's rows (the
// epoch's permutation) into the slot's pinned buffer, the copy stream moves it
// to the slot's device buffer once the step that last used the slot has
// staged it, and the compute stream waits for that copy.  The host runs up to
// kSlots steps ahead of the GPU, so the gather and the H2D overlap the
// previous steps' GEMMs and only the first copy of a call is exposed (the
// trainer synchronises once per call, not per epoch).  When a step's rows are
// consecutive in page-locked dataset memory (no shuffle), the copy stream
// reads them in place: no gather, no staging slot.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <thread>
#include <vector>

namespace lane_b200 {

struct InputPipeline {
    static constexpr int kSlots = 3;
    size_t slot_floats = 0;
    float* host[kSlots] = {};
    float* dev[kSlots] = {};
    cudaEvent_t copied[kSlots] = {};    // H2D of the slot finished (pinned buffer reusable)
    cudaEvent_t consumed[kSlots] = {};  // the step staged the slot (device buffer reusable)
    bool pending[kSlots] = {};
    cudaStream_t copy = nullptr;
    double* cum_loss_host = nullptr;  // pinned: running loss sum after every step of the call
    size_t cum_loss_count = 0;

    void reserve(size_t floats, size_t steps) {
        if (!copy) {
            LANE_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
            for (int k = 0; k < kSlots; ++k) {
                LANE_CUDA(cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
                LANE_CUDA(cudaEventCreateWithFlags(&consumed[k], cudaEventDisableTiming));
            }
        }
        if (floats > slot_floats) {
            drain();
            for (int k = 0; k < kSlots; ++k) {
                if (host[k]) LANE_CUDA(cudaFreeHost(host[k]));
                if (dev[k]) LANE_CUDA(cudaFree(dev[k]));
                host[k] = nullptr;
                dev[k] = nullptr;
                LANE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host[k]), floats * sizeof(float),
                                        cudaHostAllocDefault));
                LANE_CUDA(cudaMalloc(reinterpret_cast<void**>(&dev[k]), floats * sizeof(float)));
            }
            slot_floats = floats;
        }
        if (steps > cum_loss_count) {
            drain();
            if (cum_loss_host) LANE_CUDA(cudaFreeHost(cum_loss_host));
            cum_loss_host = nullptr;
            LANE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cum_loss_host), steps * sizeof(double),
                                    cudaHostAllocDefault));
            cum_loss_count = steps;
        }
    }
    // wait for every outstanding copy (before buffers are freed or reused)
    void drain() {
        for (int k = 0; k < kSlots; ++k)
            if (pending[k]) {
                LANE_CUDA(cudaEventSynchronize(copied[k]));
                LANE_CUDA(cudaEventSynchronize(consumed[k]));
                pending[k] = false;
            }
    }
    void release() noexcept {
        for (int k = 0; k < kSlots; ++k) {
            if (pending[k]) {
                cudaEventSynchronize(copied[k]);
                cudaEventSynchronize(consumed[k]);
            }
            if (host[k]) cudaFreeHost(host[k]);
            if (dev[k]) cudaFree(dev[k]);
            if (copied[k]) cudaEventDestroy(copied[k]);
            if (consumed[k]) cudaEventDestroy(consumed[k]);
            host[k] = dev[k] = nullptr;
            copied[k] = consumed[k] = nullptr;
            pending[k] = false;
        }
        if (cum_loss_host) cudaFreeHost(cum_loss_host);
        cum_loss_host = nullptr;
        cum_loss_count = 0;
        if (copy) cudaStreamDestroy(copy);
        copy = nullptr;
        slot_floats = 0;
    }
};

// Gather rows idx[0..rows) of X [*, F] and T [*, C] into dst = [rows][F] then
// [rows][C].  Batches over 2 MB split the rows over up to 8 host threads (the
// gather is a memory-bound copy, a few GB/s per thread).
inline void gather_rows(const float* X, const float* T, size_t F, size_t C, const uint32_t* idx, size_t rows,
                        float* dst) {
    auto part = [&](size_t r0, size_t r1) {
        for (size_t r = r0; r < r1; ++r) {
            std::memcpy(dst + r * F, X + static_cast<size_t>(idx[r]) * F, F * sizeof(float));
            std::memcpy(dst + rows * F + r * C, T + static_cast<size_t>(idx[r]) * C, C * sizeof(float));
        }
    };
    const size_t bytes = rows * (F + C) * sizeof(float);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>({bytes >> 20, static_cast<size_t>(hw), 8, rows});
    if (nt <= 1) {
        part(0, rows);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (rows + nt - 1) / nt;
    for (size_t t = 1; t < nt; ++t) {
        const size_t r0 = t * per, r1 = std::min(rows, r0 + per);
        if (r0 < r1) pool.emplace_back(part, r0, r1);
    }
    part(0, std::min(rows, per));
    for (auto& th : pool) th.join();
}

}  // namespace lane_b200
