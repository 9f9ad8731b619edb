"""Per-kernel device times of ONE mini-batch step (eager launches, no graph).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/step_c3.csv python tools/step_profile.py c3
    python tools/step_profile.py --summarize gpurun_out/step_c3.csv

Runs `warm` eager steps (LANE_B200_MB_NOGRAPH=1) and then one marked step;
the summary lists the launches of the last step in order.
"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(wl, warm=3):
    os.environ["LANE_B200_MB_NOGRAPH"] = "1"
    import bench
    from oracle import pyoracle as po
    from paper_2001_04206_b200 import lane
    F, H, C, eta, BG, mu, nb, desc = bench.MINIBATCH[wl]
    dev = lane.Device(0)
    net = lane.build_network(F, H, C, seed=42, device=dev, max_batch=BG)
    X, T = po.synthetic_dataset(F, C, BG, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    counts = []
    for _ in range(warm + 1):
        before = dev.kernel_launches
        net.minibatch_step(xd, td, BG, eta, mu)
        dev.sync()
        counts.append(dev.kernel_launches - before)
    print("launches per step", counts)


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    seq = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]
    seq.sort()
    # the step is repeated; take the last len/steps launches
    n = len(seq)
    per = int(sys.argv[3]) if len(sys.argv) > 3 else n // 4
    last = seq[-per:]
    tot = sum(v for _, _, v in last)
    print(f"| # | kernel | us | share |\n|---:|---|---:|---:|")
    for i, (_, k, v) in enumerate(last):
        print(f"| {i} | `{k[:80]}` | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    print(f"| | **step total (kernel time, serialised)** | **{tot / 1e3:.1f}** | |")


if __name__ == "__main__":
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run(sys.argv[1])
