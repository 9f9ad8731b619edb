"""Kernel-by-kernel time of one mini-batch step, measured with CUPTI through
torch.profiler (no profiler serialisation, unlike an ncu launch list), plus
the idle gaps between kernels.

    python tools/step_cupti.py [c5|c3]

Prints the top kernels (us per step, calls per step, share), the summed
kernel time per step, and the gaps before kernels.
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import pyoracle as po
from paper_2001_04206_b200 import lane, parallel
wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
F, H, C, eta, BG, mu, nb, desc = bench.MINIBATCH[wl]
dev = lane.Device(0)
net = lane.build_network(F, H, C, seed=42, device=dev, max_batch=BG)
tr = parallel.DataParallelTrainer(net, eta, mu, BG, 0, 1)
X, T = po.synthetic_dataset(F, C, nb * BG, 9)
xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
dev.h2d(xd, X); dev.h2d(td, T)
for s in range(4): tr.step(xd, td, s % nb, F, C)
dev.sync()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for s in range(5): tr.step(xd, td, s % nb, F, C)
    dev.sync()
tot = {}
for e in p.events():
    if e.device_type.name == "CUDA":
        k = e.name[:70]
        d = tot.setdefault(k, [0, 0.0]); d[0] += 1; d[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
allt = sum(v[1] for v in tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{v[1]/5:10.1f} us/step {v[0]/5:6.1f} calls/step {100*v[1]/allt:5.1f}%  {k}")
print("sum per step (us):", allt / 5)
ev = sorted([e for e in p.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
busy = 0.0; gaps = []
end = ev[0].time_range.start
for e in ev:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, e.name[:50]))
    end = max(end, e.time_range.end)
print("span per step", span / 5, "gap per step", sum(g for g, _ in gaps) / 5, "n gaps", len(gaps) / 5)
import collections
c = collections.Counter()
for g, n in gaps: c[n] += g
for n, g in c.most_common(12): print(f"  gap before {n}: {g/5:.1f} us/step")
