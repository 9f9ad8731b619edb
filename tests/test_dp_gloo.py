"""Data-parallel host logic at world size 2 on CPU (gloo).

Each rank takes its shard of the global batch (paper_2001_04206_b200.parallel.
shard_batch), computes the per-layer gradient SUMS of its rows with the oracle
(the quantity liblane_b200 all-reduces), all-reduces them with gloo, and
applies the library's update rule (g = gsum/B_global; DW = mu*DW - eta*g;
W += DW).  After several steps every rank must hold the same weights, equal
(within fp32 reassociation) to a single process stepping the full batch with
the oracle's mini-batch extension (lo_minibatch_step)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2001_04206_b200.parallel import shard_batch

F, H, C, BG, STEPS, ETA, MU = 12, [10, 7], 4, 8, 3, 0.05, 0.9


def grad_sums(net, X, T):
    from oracle import pyoracle as po
    nl = len(H) + 1
    gs = [np.zeros_like(net.get(l, po.W), dtype=np.float32) for l in range(nl)]
    bs = [np.zeros_like(net.get(l, po.B), dtype=np.float32) for l in range(nl)]
    for x, t in zip(X, T):
        net.forward(x)
        net.backward_no_update(t, ETA)
        for l in range(nl):
            d, xin = net.get(l, po.DELTAS), net.get(l, po.INPUTS)
            gs[l] += np.outer(xin, d).reshape(-1).astype(np.float32)
            bs[l] += d
    return gs, bs


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po
    X, T = po.synthetic_dataset(F, C, BG * STEPS, 3)
    net = po.OracleNet(F, H, C, seed=11)
    nl = len(H) + 1
    vW = [np.zeros_like(net.get(l, po.W)) for l in range(nl)]
    vb = [np.zeros_like(net.get(l, po.B)) for l in range(nl)]
    sh = shard_batch(BG, rank, world)
    for s in range(STEPS):
        rows = slice(s * BG + sh.begin, s * BG + sh.begin + sh.rows)
        # snapshot weights: the forward/backward of the shard must not see updates
        gs, bs = grad_sums(net, X[rows], T[rows])
        flat = torch.from_numpy(np.concatenate([np.concatenate([g, b]) for g, b in zip(gs, bs)]))
        dist.all_reduce(flat)  # the library's single allreduce of the flat gradient buffer
        flat = flat.numpy()
        invB = np.float32(1.0) / np.float32(BG)
        off = 0
        for l in range(nl):
            for buf, v in ((po.W, vW), (po.B, vb)):
                w = net.get(l, buf)
                g = flat[off:off + w.size].astype(np.float32) * invB
                off += w.size
                v[l] = np.float32(MU) * v[l] + np.float32(-ETA) * g
                net.set(l, buf, w + v[l])
    out[rank] = np.concatenate([net.get(l, po.W) for l in range(nl)])
    dist.destroy_process_group()


def test_dp_two_ranks_match_single_process_full_batch():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(worker, args=(world, port, out), nprocs=world, join=True)
    from oracle import pyoracle as po
    X, T = po.synthetic_dataset(F, C, BG * STEPS, 3)
    ref = po.OracleNet(F, H, C, seed=11)
    for s in range(STEPS):
        ref.minibatch_step(X[s * BG:(s + 1) * BG], T[s * BG:(s + 1) * BG], ETA, MU)
    want = np.concatenate([ref.get(l, po.W) for l in range(len(H) + 1)])
    np.testing.assert_array_equal(out[0], out[1])  # ranks stay in lock step
    np.testing.assert_allclose(out[0], want, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("B,world", [(4096, 8), (4096, 3), (10, 4), (8, 8)])
def test_shard_batch_partitions_the_global_batch(B, world):
    shards = [shard_batch(B, r, world) for r in range(world)]
    assert shards[0].begin == 0
    for a, b in zip(shards, shards[1:]):
        assert a.begin + a.rows == b.begin
    assert shards[-1].begin + shards[-1].rows == B
    assert max(s.rows for s in shards) - min(s.rows for s in shards) <= 1
