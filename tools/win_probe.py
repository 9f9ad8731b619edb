"""Run one windowed-SGD configuration against the oracle (debug helper).

    python tools/win_probe.py F H C n steps D [order:0/1]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    F, H, C, n, steps, D = map(int, sys.argv[1:7])
    use_order = len(sys.argv) < 8 or sys.argv[7] == "1"
    os.environ["LANE_B200_SGD_MODE"] = "window"
    os.environ["LANE_B200_SGD_WIN_D"] = str(D)
    from oracle import pyoracle as po
    from paper_2001_04206_b200 import lane
    dev = lane.Device(0)
    X, T = po.synthetic_dataset(F, C, n, 9)
    order = (np.random.default_rng(2).integers(0, n, steps) if use_order else np.arange(steps) % n).astype(np.uint32)
    net = lane.build_network(F, [H], C, seed=42, device=dev)
    orc = po.OracleNet(F, [H], C, seed=42)
    want = orc.sgd_run(X, T, steps, 0.05, order=order)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    od = 0
    if use_order:
        od = dev.alloc(order.nbytes)
        dev.h2d(od, order)
    ld = dev.alloc(8)
    dev.h2d(ld, np.zeros(1, np.float64))
    net.sgd_stream(xd, td, n, steps, 0.05, order_dev=od, loss_dev=ld)
    dev.sync()
    loss = np.zeros(1, np.float64)
    dev.d2h(loss, ld)
    w = net.hidden[0].weights
    err = np.max(np.abs(w - orc.get(0, po.W).reshape(w.shape))) / np.max(np.abs(w))
    print(f"ok F={F} H={H} C={C} n={n} steps={steps} D={D} order={use_order} loss {loss[0]:.6f} "
          f"oracle {want:.6f} W0 err {err:.2e}")


if __name__ == "__main__":
    main()
