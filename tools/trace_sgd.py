"""Per-phase cycle breakdown of the cluster SGD kernel (CTA 0, first 64 samples).

    python tools/trace_sgd.py 784x128x10
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

W0 = ["mbar wait (exchange)", "logits+softmax+d1", "hidden deltas d0", "B2 sync (pass s-1)",
      "z(s+1)+tanh", "W1 upd + partial logits", "push to peers"]


def main():
    shp = sys.argv[1] if len(sys.argv) > 1 else "784x128x10"
    F, H, C = map(int, shp.split("x"))
    path = f"/tmp/sgd_trace_{os.getpid()}.txt"
    os.environ["LANE_B200_SGD_TRACE"] = path
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
    for k in range(7):
        print(f"  warp0 {W0[k]:26s} {np.median(t[:, k + 1] - t[:, k]):7.0f} cycles")
    print(f"  warp0 loop back               {np.median(t[1:, 0] - t[:-1, 7]):7.0f}")
    print(f"  bulk  B1 -> data ready        {np.median(t[:, 9] - t[:, 8]):7.0f}")
    print(f"  bulk  pass                    {np.median(t[:, 10] - t[:, 9]):7.0f}")
    print(f"  bulk  B1(s) after warp0 d0    {np.median(t[:, 8] - t[:, 3]):7.0f}")
    print(f"  per sample                    {np.median(t[1:, 0] - t[:-1, 0]):7.0f} cycles")


if __name__ == "__main__":
    main()
