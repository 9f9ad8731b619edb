"""C5's per-rank step alone at the SCALE shard sizes (one GPU, no exchange):
ms per minibatch_step and samples/s per GPU for each batch given.

    python tools/shard_step.py 4096 2048 1024 512
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import pyoracle as po
from paper_2001_04206_b200 import lane
F, H, C = 4096, [4096] * 8, 10
dev = lane.Device(0)
stream = torch.cuda.ExternalStream(dev.stream)
for B in [int(x) for x in sys.argv[1:]]:
    net = lane.build_network(F, H, C, seed=42, device=dev, max_batch=B)
    X, T = po.synthetic_dataset(F, C, 4 * B, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X); dev.h2d(td, T)
    for s in range(4): net.minibatch_step(xd + (s % 4) * B * F * 4, td + (s % 4) * B * C * 4, B, 1e-3, 0.0)
    dev.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(20): net.minibatch_step(xd + (s % 4) * B * F * 4, td + (s % 4) * B * C * 4, B, 1e-3, 0.0)
    e1.record(stream); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"B={B}: {ms:.3f} ms/step, {B / ms * 1e3:.0f} samples/s per GPU")
    dev.free(xd); dev.free(td); net.close()
