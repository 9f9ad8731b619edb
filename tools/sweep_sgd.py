"""Sweep the fused online-SGD kernel over CTA counts / shapes (device-timed).

    python tools/sweep_sgd.py --shapes 784x128x10,340x1024x10 --ctas 8,16,32,64,128
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="784x128x10")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--samples", type=int, default=20000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="auto")
    args = ap.parse_args()
    import torch
    from oracle import pyoracle as po
    from paper_2001_04206_b200 import lane
    dev = lane.Device(0)
    stream = torch.cuda.ExternalStream(dev.stream)
    for shp in args.shapes.split(","):
        F, H, C = map(int, shp.split("x"))
        n = args.samples
        X, T = po.synthetic_dataset(F, C, min(n, 4096), 9)
        xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
        dev.h2d(xd, X)
        dev.h2d(td, T)
        for mode in args.modes.split(","):
          for g in args.ctas.split(","):
            for k in ("LANE_B200_SGD_CTAS", "LANE_B200_SGD_CLUSTER", "LANE_B200_SGD_MODE",
                      "LANE_B200_SGD_STREAM"):
                os.environ.pop(k, None)
            if mode != "auto":
                os.environ["LANE_B200_SGD_MODE"] = "grid" if mode == "stream" else mode
            if mode == "stream":
                os.environ["LANE_B200_SGD_STREAM"] = "1"
            if g != "0":
                os.environ["LANE_B200_SGD_CLUSTER" if mode == "cluster" else "LANE_B200_SGD_CTAS"] = g
            net = lane.build_network(F, [H], C, seed=42, device=dev)
            net.sgd_stream(xd, td, len(X), 2000, 0.01)
            dev.sync()
            best = 1e30
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                net.sgd_stream(xd, td, len(X), n, 0.01)
                e1.record(stream)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(json.dumps({"shape": shp, "mode": mode, "ctas": g, "us_per_sample": 1000 * best / n,
                              "samples_per_s": n / (best / 1000)}), flush=True)
            net.close()
        dev.free(xd)
        dev.free(td)


if __name__ == "__main__":
    main()
