"""Per-phase cycle breakdown of the windowed SGD kernel's chain CTA
(first 64 samples of a 512-sample stream; the second call is measured).

    python tools/trace_window.py 784x128x10 [D]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PH = ["z + tanh + W1 update(s-1) + W1.t", "partial logits + reduce", "softmax/E + d0",
      "publish d0", "off-chain (p, d1, biases, shift)", "fetch row s+1"]


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
    rows = int(os.environ.get("TRACE_ROWS", "512"))
    steps = int(os.environ.get("TRACE_STEPS", "512"))
    X, T = po.synthetic_dataset(F, C, rows, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    net = lane.build_network(F, [H], C, seed=42, device=dev)
    net.sgd_stream(xd, td, rows, steps, 0.01)
    net.sgd_stream(xd, td, rows, steps, 0.01)
    dev.sync()
    lines = open(path).read().strip().splitlines()
    print(shp, lines[-65])
    T_ = np.array([[int(v) for v in ln.split()] for ln in lines[-64:]], dtype=np.int64)
    t = T_[8:]

    def row(name, d):
        d = np.asarray(d)
        print(f"  {name:34s} median {np.median(d):7.0f}  mean {np.mean(d):7.0f}  max {np.max(d):7.0f}")
    row("  z + tanh (of phase 0)", t[:, 14] - t[:, 0])
    row("  flag wait + fetch row s+1", t[:, 15] - t[:, 14])
    row("  W1 update (s-1)", t[:, 1] - t[:, 15])
    for k in range(len(PH)):
        row(PH[k], t[:, k + 1] - t[:, k])
    row("loop back", t[1:, 0] - t[:-1, 6])
    row("per sample", t[1:, 0] - t[:-1, 0])
    # helper slack: flag of row r set at T_[r,7]; chain fetches row r at T_[r-1,5]
    r = np.arange(9, 64)
    row("helper slack (flag before fetch)", T_[r - 1, 5] - T_[r, 7])
    row("helper wake after publish", t[:, 12] - t[:, 4])
    row("helper rows pass", t[:, 13] - t[:, 12])
    row("helper done before next publish", t[1:, 4] - t[:-1, 13])
    for b in (1, 2, 3):
        s0 = 16 * b
        print(f"  block {b}: loader wait {T_[s0, 9] - T_[s0, 8]:6d}  stage {T_[s0, 10] - T_[s0, 9]:6d}  "
              f"ready-before-need {T_[s0 - 1, 5] - T_[s0, 10]:7d}  | publisher: after block end "
              f"{T_[s0, 11] - T_[s0 + 15, 4]:6d}  publish {T_[s0 + 1, 11] - T_[s0, 11]:6d}  "
              f"stats {T_[s0 + 2, 11] - T_[s0 + 1, 11]:6d}")


if __name__ == "__main__":
    main()
