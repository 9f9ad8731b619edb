// Input side of the path: the reference's dataset functions
// (include/lane/dataset.hpp, src/dataset.cpp) as host code in the library, with
// the rows kept in page-locked memory so every host->device copy of a batch
// runs at full PCIe/C2C rate and overlaps the step (see pipeline.cuh).
//
// Layout: one allocation, X [n][feature_width] then T [n][class_count],
// row-major fp32 -- the exact layout lane_b200_train / _train_minibatch read.
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <system_error>
#include <vector>

struct lane_b200_dataset {
    size_t features = 0, classes = 0, n = 0;
    float* X = nullptr;  // n * features, then T = X + n * features
    float* T = nullptr;
    bool pinned = false;

    ~lane_b200_dataset() { release(); }
    void release() {
        if (X) {
            if (pinned)
                cudaFreeHost(X);
            else
                std::free(X);
        }
        X = T = nullptr;
        n = 0;
    }
    // Page-locked when a CUDA device is present (the staging the batch
    // pipeline copies from); plain memory otherwise (host-only use).
    void allocate(size_t F, size_t C, size_t rows) {
        release();
        features = F;
        classes = C;
        n = rows;
        const size_t bytes = std::max<size_t>(rows * (F + C), 1) * sizeof(float);
        int ndev = 0;
        void* p = nullptr;
        if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 &&
            cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
            pinned = true;
        } else {
            cudaGetLastError();  // clear the no-device error
            p = std::malloc(bytes);
            pinned = false;
            if (!p) throw Error(LANE_ERR_INTERNAL, "dataset: out of host memory");
        }
        X = static_cast<float*>(p);
        T = X + rows * F;
    }
};

namespace lane_b200 {
namespace dataset {

// dataset.cpp:18-27: std::from_chars over the whole field (no leading '+' or
// blanks, trailing characters rejected), correctly rounded to float.
inline float parse_field(const char* first, const char* last, size_t line_no) {
    float value = 0.0f;
    const auto res = std::from_chars(first, last, value);
    if (res.ec != std::errc() || res.ptr != last)
        throw Error(LANE_ERR_PARSE, "line " + std::to_string(line_no) + ": bad numeric field '" +
                                        std::string(first, last) + "'");
    return value;
}

// load_dataset (dataset.cpp:31-83).  The file is read whole; lines split on
// '\n' with one trailing '\r' dropped; empty lines skipped; fields split on
// ',' exactly as std::getline(ss, field, ',') does (a trailing ',' adds no
// empty field, an inner ",," does).
inline void load(const char* path, size_t F, size_t C, lane_b200_dataset& d) {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw Error(LANE_ERR_IO, std::string("cannot open dataset file: ") + path);
    std::string buf;
    {
        char chunk[1 << 16];
        size_t got;
        while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.append(chunk, got);
        std::fclose(f);
    }
    const size_t want = F + C;
    std::vector<float> X, T;
    std::vector<std::pair<const char*, const char*>> fields;
    size_t line_no = 0, pos = 0;
    while (pos < buf.size()) {
        size_t end = buf.find('\n', pos);
        if (end == std::string::npos) end = buf.size();
        const char* b = buf.data() + pos;
        const char* e = buf.data() + end;
        pos = end + 1;
        ++line_no;
        if (e > b && e[-1] == '\r') --e;
        if (e == b) continue;
        fields.clear();
        const char* s = b;
        while (s < e) {
            const char* c = static_cast<const char*>(std::memchr(s, ',', static_cast<size_t>(e - s)));
            if (!c) {
                fields.emplace_back(s, e);
                break;
            }
            fields.emplace_back(s, c);
            s = c + 1;
        }
        if (fields.size() != want)
            throw Error(LANE_ERR_PARSE, "line " + std::to_string(line_no) + ": expected " + std::to_string(want) +
                                            " fields, got " + std::to_string(fields.size()));
        for (size_t i = 0; i < F; ++i) X.push_back(parse_field(fields[i].first, fields[i].second, line_no));
        size_t ones = 0;
        for (size_t c = 0; c < C; ++c) {
            const float v = parse_field(fields[F + c].first, fields[F + c].second, line_no);
            if (v != 0.0f && v != 1.0f)
                throw Error(LANE_ERR_PARSE, "line " + std::to_string(line_no) + ": label field must be 0 or 1");
            if (v == 1.0f) ++ones;
            T.push_back(v);
        }
        if (ones != 1) throw Error(LANE_ERR_PARSE, "line " + std::to_string(line_no) + ": label is not one-hot");
    }
    const size_t n = F ? X.size() / F : T.size() / std::max<size_t>(C, 1);
    d.allocate(F, C, n);
    if (!X.empty()) std::memcpy(d.X, X.data(), X.size() * sizeof(float));
    if (!T.empty()) std::memcpy(d.T, T.data(), T.size() * sizeof(float));
}

// save_dataset (dataset.cpp:85-103): features at %.9g (round-trips fp32),
// labels written as '1' / '0'.
inline void save(const lane_b200_dataset& d, const char* path) {
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(LANE_ERR_IO, std::string("cannot write dataset file: ") + path);
    std::string line;
    char tmp[64];
    for (size_t r = 0; r < d.n; ++r) {
        line.clear();
        for (size_t i = 0; i < d.features; ++i) {
            std::snprintf(tmp, sizeof tmp, "%.9g", static_cast<double>(d.X[r * d.features + i]));
            line += tmp;
            line += ',';
        }
        for (size_t c = 0; c < d.classes; ++c) {
            line += d.T[r * d.classes + c] == 1.0f ? '1' : '0';
            line += c + 1 < d.classes ? ',' : '\n';
        }
        if (std::fwrite(line.data(), 1, line.size(), f) != line.size()) {
            std::fclose(f);
            throw Error(LANE_ERR_IO, std::string("cannot write dataset file: ") + path);
        }
    }
    std::fclose(f);
}

inline void copy_row(const lane_b200_dataset& s, size_t r, lane_b200_dataset& d, size_t at) {
    std::memcpy(d.X + at * d.features, s.X + r * s.features, s.features * sizeof(float));
    std::memcpy(d.T + at * d.classes, s.T + r * s.classes, s.classes * sizeof(float));
}

// split (dataset.cpp:105-124): Fisher-Yates over iota with SeededRng(seed),
// the first floor(frac * n) permuted items train, the rest test.
inline void split(const lane_b200_dataset& d, double frac, uint64_t seed, lane_b200_dataset& train,
                  lane_b200_dataset& test) {
    if (!(frac > 0.0 && frac < 1.0)) throw Error(LANE_ERR_CONFIG, "split: train_fraction must be in (0, 1)");
    std::vector<size_t> order(d.n);
    for (size_t i = 0; i < d.n; ++i) order[i] = i;
    SplitMix64 rng(seed);
    for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[rng.below(i)]);
    const size_t n_train = static_cast<size_t>(std::floor(frac * static_cast<double>(d.n)));
    train.allocate(d.features, d.classes, n_train);
    test.allocate(d.features, d.classes, d.n - n_train);
    for (size_t k = 0; k < d.n; ++k) {
        if (k < n_train)
            copy_row(d, order[k], train, k);
        else
            copy_row(d, order[k], test, k - n_train);
    }
}

// enlarge (dataset.cpp:126-148): factor copies of each item in order; with
// noise > 0 every feature becomes clamp(x + rng.uniform(-noise, noise), 0, 1).
// rng_state is the SeededRng's state, advanced in place.
inline void enlarge(const lane_b200_dataset& d, size_t factor, float noise, uint64_t& rng_state,
                    lane_b200_dataset& out) {
    if (factor == 0) throw Error(LANE_ERR_CONFIG, "enlarge: factor must be >= 1");
    if (noise < 0.0f) throw Error(LANE_ERR_CONFIG, "enlarge: noise must be non-negative");
    SplitMix64 rng(rng_state);
    out.allocate(d.features, d.classes, d.n * factor);
    size_t at = 0;
    for (size_t r = 0; r < d.n; ++r) {
        for (size_t k = 0; k < factor; ++k, ++at) {
            copy_row(d, r, out, at);
            if (noise > 0.0f) {
                float* x = out.X + at * out.features;
                for (size_t i = 0; i < out.features; ++i) x[i] = std::clamp(x[i] + rng.uniform(-noise, noise), 0.0f, 1.0f);
            }
        }
    }
    rng_state = rng.state;
}

}  // namespace dataset
}  // namespace lane_b200
