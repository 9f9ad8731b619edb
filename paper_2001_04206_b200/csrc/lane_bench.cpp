// lane-bench for the B200 path: the reference's benchmark harness
// (proj/tools/lane_bench.cpp, proj/src/bench.cpp run_benchmark/emit_report)
// with a "b200" device.  Same flags, same measurement protocol (warm-up
// executions, then the arithmetic mean of the timed ones; each iteration one
// sample end to end: forward, then BackwardPlan::run), same report columns
// kernel,device,mean_ms,copy_in_ms,kernel_ms,copy_out_ms,speedup.
//
// The per-kernel split comes from BackwardPlan::run's PhaseTiming (CUDA
// events around each schedule).  The reference's serial/parallel rows are
// produced by the reference's own lane-bench; pass its CSV with
// --baseline-csv and the b200 rows are appended with speedup = serial mean /
// b200 mean, i.e. the paper's per-kernel table with a B200 column.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "lane_b200/lane.hpp"

using namespace lane_b200;

namespace {

struct Config {
    std::string dataset;
    std::size_t features = 4, classes = 3, fc_neurons = 8;
    float eta = 0.01f;
    std::size_t warmup = 10000, iters = 10, enlarge = 1;
    std::string device = "b200";
    unsigned workers = 0;
    std::uint64_t seed = 42;
    std::string format = "csv", out, baseline_csv;
    bool print_hash = false;
    bool strict = false;
};

struct Row {
    std::string kernel, device;
    double mean_ms = 0, copy_in_ms = 0, kernel_ms = 0, copy_out_ms = 0, speedup = 1;
};

const char* kUsage =
    "lane-bench (B200): backward-kernel timing harness\n"
    "  --dataset PATH        delimited dataset file (required)\n"
    "  --features N          input feature count (4)\n"
    "  --classes N           output class count (3)\n"
    "  --fc-neurons N        neurons in the fully connected layer (8)\n"
    "  --eta X               learning rate (0.01)\n"
    "  --warmup N            unmeasured warm-up executions (10000)\n"
    "  --iters N             timed iterations averaged into the report (10)\n"
    "  --enlarge N           replicate each sample this many times (1)\n"
    "  --device b200         device under test (serial/parallel are the reference's CPU backends)\n"
    "  --workers N           accepted for compatibility (CPU worker count)\n"
    "  --seed N              seed for weights and enlargement (42)\n"
    "  --format csv|md       report format (csv)\n"
    "  --out PATH            write the report here instead of stdout\n"
    "  --baseline-csv PATH   the reference lane-bench CSV to merge (speedup vs its serial rows)\n"
    "  --numerics fast|strict  strict = the reference's rounding and order, bit-identical weights (fast)\n"
    "  --print-hash          print the final weights hash (FNV-1a, bench.cpp:32-41) on stderr\n";

struct ConfigError2 : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class T>
T parse_num(const std::string& flag, const std::string& v) {
    // unsigned options: "-1" would wrap to a huge count (CLI11 rejects it)
    if (std::is_unsigned<T>::value && v.find('-') != std::string::npos)
        throw ConfigError2(flag + ": bad value '" + v + "'");
    std::istringstream is(v);
    T x{};
    is >> x;
    if (!is || !is.eof()) throw ConfigError2(flag + ": bad value '" + v + "'");
    return x;
}

Config parse(int argc, char** argv) {
    Config c;
    bool have_dataset = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i], v;
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
            v = a.substr(eq + 1);
            a = a.substr(0, eq);
        }
        auto val = [&]() -> std::string {
            if (eq != std::string::npos) return v;
            if (i + 1 >= argc) throw ConfigError2(a + ": missing value");
            return argv[++i];
        };
        if (a == "-h" || a == "--help") {
            std::cout << kUsage;
            std::exit(0);
        } else if (a == "--dataset") {
            c.dataset = val();
            have_dataset = true;
        } else if (a == "--features") {
            c.features = parse_num<std::size_t>(a, val());
        } else if (a == "--classes") {
            c.classes = parse_num<std::size_t>(a, val());
        } else if (a == "--fc-neurons") {
            c.fc_neurons = parse_num<std::size_t>(a, val());
        } else if (a == "--eta") {
            c.eta = parse_num<float>(a, val());
        } else if (a == "--warmup") {
            c.warmup = parse_num<std::size_t>(a, val());
        } else if (a == "--iters") {
            c.iters = parse_num<std::size_t>(a, val());
        } else if (a == "--enlarge") {
            c.enlarge = parse_num<std::size_t>(a, val());
        } else if (a == "--device") {
            c.device = val();
        } else if (a == "--workers") {
            c.workers = parse_num<unsigned>(a, val());
        } else if (a == "--seed") {
            c.seed = parse_num<std::uint64_t>(a, val());
        } else if (a == "--format") {
            c.format = val();
        } else if (a == "--out") {
            c.out = val();
        } else if (a == "--baseline-csv") {
            c.baseline_csv = val();
        } else if (a == "--numerics") {
            const std::string m = val();
            if (m != "strict" && m != "fast") throw ConfigError2("--numerics must be 'strict' or 'fast'");
            c.strict = m == "strict";
        } else if (a == "--print-hash") {
            c.print_hash = true;
        } else {
            throw ConfigError2("unknown option " + a);
        }
    }
    if (!have_dataset) throw ConfigError2("--dataset is required");
    if (c.device != "b200")
        throw ConfigError2("--device must be 'b200' (run the reference's lane-bench for '" + c.device +
                           "' and merge its CSV with --baseline-csv)");
    if (c.format != "csv" && c.format != "md") throw ConfigError2("--format must be 'csv' or 'md'");
    // run_benchmark's checks (bench.cpp:152-161)
    if (c.iters == 0) throw ConfigError2("benchmark: timed_iters must be >= 1");
    if (c.features == 0 || c.fc_neurons == 0 || c.classes < 2)
        throw ConfigError2("benchmark: invalid network topology");
    if (!(c.eta > 0.0f)) throw ConfigError2("benchmark: eta must be positive");
    return c;
}

// SeededRng(seed).split() (tensor.hpp:40): the child's seed is the parent's
// first draw xor the golden-ratio constant.
std::uint64_t split_seed(std::uint64_t seed) {
    std::uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return (z ^ (z >> 31)) ^ 0x9E3779B97F4A7C15ULL;
}

std::vector<Row> read_baseline(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError2("cannot read --baseline-csv " + path);
    std::vector<Row> rows;
    std::string line;
    bool header = true;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (header) {
            header = false;
            if (line.rfind("kernel,device,", 0) == 0) continue;
        }
        std::vector<std::string> f;
        std::stringstream ss(line);
        std::string x;
        while (std::getline(ss, x, ',')) f.push_back(x);
        if (f.size() != 7) throw ConfigError2("--baseline-csv: expected 7 columns: " + line);
        Row r;
        r.kernel = f[0];
        r.device = f[1];
        r.mean_ms = std::atof(f[2].c_str());
        r.copy_in_ms = std::atof(f[3].c_str());
        r.kernel_ms = std::atof(f[4].c_str());
        r.copy_out_ms = std::atof(f[5].c_str());
        r.speedup = std::atof(f[6].c_str());
        rows.push_back(r);
    }
    return rows;
}

std::string emit(const std::vector<Row>& rows, const std::string& format) {
    std::ostringstream out;
    char buf[200];
    if (format == "csv") {
        out << "kernel,device,mean_ms,copy_in_ms,kernel_ms,copy_out_ms,speedup\n";
        for (const Row& r : rows) {
            std::snprintf(buf, sizeof buf, "%s,%s,%.3f,%.3f,%.3f,%.3f,%.3f\n", r.kernel.c_str(), r.device.c_str(),
                          r.mean_ms, r.copy_in_ms, r.kernel_ms, r.copy_out_ms, r.speedup);
            out << buf;
        }
        return out.str();
    }
    out << "| kernel | device | mean_ms | copy_in_ms | kernel_ms | copy_out_ms | speedup |\n";
    out << "|---|---|---|---|---|---|---|\n";
    for (const Row& r : rows) {
        std::snprintf(buf, sizeof buf, "| %s | %s | %.3f | %.3f | %.3f | %.3f | %.3f |\n", r.kernel.c_str(),
                      r.device.c_str(), r.mean_ms, r.copy_in_ms, r.kernel_ms, r.copy_out_ms, r.speedup);
        out << buf;
    }
    return out.str();
}

}  // namespace

int main(int argc, char** argv) {
    Config cfg;
    std::vector<Row> baseline;
    try {
        cfg = parse(argc, argv);
        if (!cfg.baseline_csv.empty()) baseline = read_baseline(cfg.baseline_csv);
    } catch (const std::exception& e) {
        std::cerr << "configuration error: " << e.what() << "\n" << kUsage;
        return 2;
    }
    try {
        DataSet ds = load_dataset(cfg.dataset, cfg.features, cfg.classes);
        if (cfg.enlarge > 1) {
            SeededRng rng(split_seed(cfg.seed));
            ds = enlarge(ds, cfg.enlarge, 0.01f, rng);
        }
        if (ds.size() == 0) throw ConfigError("benchmark: dataset has no samples");

        Device dev(0, cfg.strict ? Numerics::Strict : Numerics::Fast);
        auto net = build_network(dev, cfg.features, {cfg.fc_neurons}, cfg.classes, cfg.seed);
        BackwardPlan plan(*net, LearningRate(cfg.eta));
        const std::size_t F = cfg.features, C = cfg.classes;
        std::vector<float> x(F), t(C);
        double sum[2][3] = {};
        for (std::size_t it = 0; it < cfg.warmup + cfg.iters; ++it) {
            const std::size_t k = it % ds.size();
            x.assign(ds.features.begin() + k * F, ds.features.begin() + (k + 1) * F);
            t.assign(ds.labels.begin() + k * C, ds.labels.begin() + (k + 1) * C);
            net->forward(x);
            const std::vector<PhaseTiming> tm = plan.run(t);
            if (it >= cfg.warmup)
                for (int r = 0; r < 2; ++r) {
                    sum[r][0] += tm[r].copy_in_ms;
                    sum[r][1] += tm[r].kernel_ms;
                    sum[r][2] += tm[r].copy_out_ms;
                }
        }
        const char* names[2] = {"softmax_backward", "fc_backward"};
        std::map<std::string, double> serial_mean;
        for (const Row& r : baseline)
            if (r.device == "serial") serial_mean[r.kernel] = r.mean_ms;
        std::vector<Row> rows;
        for (int r = 0; r < 2; ++r) {
            for (const Row& b : baseline)
                if (b.kernel == names[r]) rows.push_back(b);
            Row m;
            m.kernel = names[r];
            m.device = "b200";
            m.copy_in_ms = sum[r][0] / static_cast<double>(cfg.iters);
            m.kernel_ms = sum[r][1] / static_cast<double>(cfg.iters);
            m.copy_out_ms = sum[r][2] / static_cast<double>(cfg.iters);
            m.mean_ms = m.copy_in_ms + m.kernel_ms + m.copy_out_ms;
            const auto s = serial_mean.find(names[r]);
            m.speedup = s != serial_mean.end() && m.mean_ms > 0 ? s->second / m.mean_ms : std::nan("");
            rows.push_back(m);
        }
        const std::string text = emit(rows, cfg.format);
        if (cfg.out.empty()) {
            std::cout << text;
        } else {
            std::ofstream out(cfg.out);
            if (!out) {
                std::cerr << "error: cannot write " << cfg.out << "\n";
                return 1;
            }
            out << text;
        }
        if (cfg.print_hash) std::fprintf(stderr, "final_weights_hash=%016llx\n", (unsigned long long)net->hash());
        return 0;
    } catch (const ConfigError& e) {
        std::cerr << "configuration error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
