// Exhaustive host check of paper_2001_04206_b200/csrc/lane_libm.cuh against the
// running glibc: every float bit pattern in [lo, hi) (as uint32) for tanhf,
// expf and logf.  Prints mismatch counts and the first few mismatches.
// Build: g++ -O2 -ffp-contract=off -fopenmp (no -march: no FMA contraction).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../paper_2001_04206_b200/csrc/lane_libm.cuh"

static float bits2f(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }
static uint32_t f2bits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }

template <class F, class G>
static long check(const char* name, F mine, G ref, uint64_t lo, uint64_t hi, uint64_t stride) {
    long bad = 0;
#pragma omp parallel for reduction(+ : bad) schedule(static, 1 << 16)
    for (int64_t u = (int64_t)lo; u < (int64_t)hi; u += (int64_t)stride) {
        const float x = bits2f((uint32_t)u);
        const float a = mine(x), b = ref(x);
        const bool same = (std::isnan(a) && std::isnan(b)) || f2bits(a) == f2bits(b);
        if (!same) {
            if (bad < 5) {
#pragma omp critical
                std::printf("  %s(%a) mine %a glibc %a\n", name, x, a, b);
            }
            ++bad;
        }
    }
    std::printf("%s: %ld mismatches over [%#llx, %#llx) stride %llu\n", name, bad,
                (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)stride);
    return bad;
}

int main(int argc, char** argv) {
    const uint64_t stride = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1;
    long bad = 0;
    auto t_m = [](float x) { return lane_libm::tanhf(x); };
    auto t_r = [](float x) { return ::tanhf(x); };
    auto e_m = [](float x) { return lane_libm::expf(x); };
    auto e_r = [](float x) { return ::expf(x); };
    auto l_m = [](float x) { return lane_libm::logf(x); };
    auto l_r = [](float x) { return ::logf(x); };
    bad += check("tanhf", t_m, t_r, 0, 1ull << 32, stride);
    bad += check("expf", e_m, e_r, 0, 1ull << 32, stride);
    bad += check("logf", l_m, l_r, 0, 1ull << 32, stride);
    std::printf("TOTAL_MISMATCHES %ld\n", bad);
    return bad ? 1 : 0;
}
