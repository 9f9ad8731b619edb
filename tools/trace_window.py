"""Per-phase cycle breakdown of the windowed SGD kernel's critical warp
(first 64 samples of a 512-sample stream; the second call is measured).

    python tools/trace_window.py 784x128x10 [D]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PH = ["waits (Y block, row ready)", "z + tanh", "partial logits + reduce", "softmax + d1 bcast",
      "d0 + publish"]


def main():
    shp = sys.argv[1] if len(sys.argv) > 1 else "784x128x10"
    F, H, C = map(int, shp.split("x"))
    if len(sys.argv) > 2:
        os.environ["LANE_B200_SGD_WIN_D"] = sys.argv[2]
    path = f"/tmp/win_trace_{os.getpid()}.txt"
    os.environ["LANE_B200_SGD_TRACE"] = path
    os.environ.setdefault("LANE_B200_SGD_MODE", "window")
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
    t = np.array([[int(v) for v in ln.split()] for ln in lines[-64:]], dtype=np.int64)[8:]
    def row(name, d):
        print(f"  {name:28s} median {np.median(d):7.0f}  mean {np.mean(d):7.0f}  max {np.max(d):7.0f}")
    for k in range(len(PH)):
        row(PH[k], t[:, k + 1] - t[:, k])
    row("tail + loop back", t[1:, 0] - t[:-1, len(PH)])
    row("per sample", t[1:, 0] - t[:-1, 0])


if __name__ == "__main__":
    main()
