"""Generate tests/golden/lane_bench.json from the UNMODIFIED reference's
lane::run_benchmark (proj/src/bench.cpp:147-185) through oracle/_ref:

    make -C oracle && python tests/golden/make_lane_bench_golden.py

Each entry is a lane-bench configuration on the Iris fixture and the
reference's BenchReport.final_weights_hash (FNV-1a over every layer's weights
and biases after warmup + iters samples of forward + BackwardPlan::run).  The
B200 lane-bench (paper_2001_04206_b200/lib/lane-bench --numerics strict
--print-hash) must print the same hash (tests/test_lane_bench.py).
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402

CONFIGS = [  # fc_neurons, eta, warmup, iters, enlarge, seed
    (8, 0.01, 200, 10, 1, 42),
    (8, 0.01, 100, 10, 3, 42),
    (32, 0.05, 300, 20, 1, 42),
    (16, 0.1, 50, 5, 2, 7),
]


def main():
    f = po.ref_lib().lr_run_benchmark
    f.restype = C.c_long
    f.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float, C.c_size_t, C.c_size_t,
                  C.c_size_t, C.c_int, C.c_uint, C.c_uint64, C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64)]
    iris = os.path.join(HERE, "iris_normalized.txt").encode()
    out = []
    for fc, eta, warm, iters, enl, seed in CONFIGS:
        buf, h = C.create_string_buffer(4096), C.c_uint64()
        assert f(iris, 4, 3, fc, eta, warm, iters, enl, 0, 1, seed, buf, 4096, C.byref(h)) > 0
        out.append({"fc_neurons": fc, "eta": eta, "warmup": warm, "iters": iters, "enlarge": enl,
                    "seed": seed, "final_weights_hash": f"{h.value:016x}"})
    with open(os.path.join(HERE, "lane_bench.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
