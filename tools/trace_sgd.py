"""Per-phase cycle breakdown of the fused SGD kernel (CTA 0, first 64 samples).

    python tools/trace_sgd.py 784x128x10 [cluster|grid]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = ["prefetch+wait+sync", "forward dot+sync", "tanh+sync", "partial logits+sync",
          "push partials", "cluster barrier", "softmax/deltas/loss"]


def main():
    shp = sys.argv[1] if len(sys.argv) > 1 else "784x128x10"
    mode = sys.argv[2] if len(sys.argv) > 2 else "cluster"
    F, H, C = map(int, shp.split("x"))
    path = f"/tmp/sgd_trace_{os.getpid()}.txt"
    os.environ["LANE_B200_SGD_TRACE"] = path
    os.environ["LANE_B200_SGD_MODE"] = mode
    from oracle import pyoracle as po
    from paper_2001_04206_b200 import lane
    dev = lane.Device(0)
    X, T = po.synthetic_dataset(F, C, 512, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    net = lane.build_network(F, [H], C, seed=42, device=dev)
    net.sgd_stream(xd, td, 512, 512, 0.01)
    net.sgd_stream(xd, td, 512, 512, 0.01)
    dev.sync()
    lines = open(path).read().strip().splitlines()
    print(shp, lines[-65])
    t = np.array([[int(v) for v in ln.split()] for ln in lines[-64:]], dtype=np.int64)
    t = t[8:]  # skip warm-up samples
    d = np.diff(t, axis=1)
    for k in range(7):
        print(f"  {PHASES[k]:24s} median {np.median(d[:, k]):8.0f} cycles")
    print(f"  {'loop back':24s} median {np.median(t[1:, 0] - t[:-1, 7]):8.0f} cycles")
    print(f"  per sample: {np.median(t[1:, 0] - t[:-1, 0]):.0f} cycles")


if __name__ == "__main__":
    main()
