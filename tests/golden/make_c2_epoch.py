"""Generate tests/golden/c2_epoch.npz: one 60,000-sample epoch of the bench's
C2 workload (784-128-10, online SGD, eta = 0.01) through the UNMODIFIED
reference (oracle/_ref/liblane_ref.so: proj/src/*.cpp, Release flags, driven
through lane::train, proj/src/network.cpp:140-182).

    make -C oracle && python tests/golden/make_c2_epoch.py

Inputs are regenerated on any machine: features U[0,1) and one-hot labels
from SeededRng(9) exactly as testsupport::synthetic_dataset
(proj/tests/test_support.hpp:14-27), weights from build_network(seed 42),
TrainerConfig(eta 0.01, max_error 0, 1 epoch, shuffle seed 42).  The fixture
holds the epoch's EpochStats and the final weights and biases of both
layers, plus the reference's FNV-1a weight hash (proj/src/bench.cpp:32-41).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402

F, H, C, N, ETA, SEED_DATA, SEED_NET, SEED_SHUFFLE = 784, 128, 10, 60000, 0.01, 9, 42, 42


def main():
    X, T = po.synthetic_dataset(F, C, N, SEED_DATA)
    net = po.RefNet(F, [H], C, seed=SEED_NET)
    t0 = time.time()
    stats = net.train(X, T, ETA, max_epochs=1, max_error=0.0, seed=SEED_SHUFFLE)
    print(f"reference epoch: {time.time() - t0:.1f} s, stats {stats}")
    (_, loss, acc), = stats
    out = {
        "config": np.array([F, H, C, N, SEED_DATA, SEED_NET, SEED_SHUFFLE], np.int64),
        "eta": np.float32(ETA),
        "mean_loss": np.float32(loss),
        "accuracy": np.float32(acc),
        "hash": np.uint64(net.hash()),
    }
    for l in range(2):
        out[f"W{l}"] = net.get(l, po.W)
        out[f"b{l}"] = net.get(l, po.B)
    np.savez_compressed(os.path.join(HERE, "c2_epoch.npz"), **out)


if __name__ == "__main__":
    main()
