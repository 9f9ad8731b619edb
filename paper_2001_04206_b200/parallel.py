"""Data-parallel mini-batch training -- host-side driver.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing only:
rank 0 creates the NCCL unique id inside liblane_b200 and broadcasts it; every
rank binds its lane context to the communicator (``lane_b200_comm_init``).
Each step a rank runs forward/dgrad/wgrad on its shard of the global batch.
The library all-reduces (NCCL fp32 sum) each layer's span of the flat gradient
buffer (G and bias gradients, contiguous per layer in HBM) as soon as that
layer's wgrad is done -- one allreduce per layer, in reverse layer order, on a
communication stream that overlaps the rest of the backward -- and then every
rank applies the identical update, with 1/B_global folded into the step:

    G = (1/B_global) * sum_{ranks} sum_{b in shard} delta_b (x) x_b
    DW = mu*DW + (-eta)*G ;  W += DW

With NVLS (``init_nvls``: the arena bound to an NVSwitch multicast object) the
exchange is fused with the update instead: each rank reduces its slice of the
gradient sums through the switch, updates it and multicasts W, the velocities
and the mean gradients back to every rank (csrc/nvls.cuh).

Batch-1 online SGD (configs C1, C2, C4) has a strict sample-to-sample
dependency and does not shard: N GPUs run N independent replicas.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    begin: int  # first row of the global batch owned by this rank
    rows: int   # rows owned by this rank


def shard_batch(global_batch: int, rank: int, world: int) -> Shard:
    """Contiguous, balanced split of a global batch (rows differ by at most 1).
    Ranks own consecutive row ranges in rank order, so the union over ranks is
    the global batch in its original order."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if global_batch < world:
        raise ValueError("global batch smaller than the number of ranks")
    base, extra = divmod(global_batch, world)
    rows = base + (1 if rank < extra else 0)
    begin = rank * base + min(rank, extra)
    return Shard(rank, world, begin, rows)


def init_comm(device, rank: int, world: int, group=None) -> None:
    """Bind ``device`` (a lane.Device) to an NCCL communicator of ``world``
    ranks.  Uses torch.distributed (any backend) only to broadcast the id."""
    import torch.distributed as dist
    uid = [device.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    device.comm_init(rank, world, uid[0])


def _fd_socket_path(tag: str) -> str:
    return "\0lane_b200_nvls_" + tag  # Linux abstract socket namespace


def exchange_fd(fd: int, rank: int, world: int, tag: str, timeout: float = 60.0) -> int:
    """Rank 0 sends the open file descriptor ``fd`` to ranks 1..world-1 over a
    Unix-domain socket (SCM_RIGHTS); every other rank returns its received copy.
    ``tag`` must be unique per job (the socket lives in the abstract namespace)."""
    import socket
    import time
    path = _fd_socket_path(tag)
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path)
        srv.listen(world)
        srv.settimeout(timeout)
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"F"], [fd])
                    conn.recv(1)  # the peer holds its copy: safe to close ours later
        finally:
            srv.close()
        return fd
    deadline = time.time() + timeout
    while True:
        try:
            cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            cli.connect(path)
            break
        except (FileNotFoundError, ConnectionRefusedError):
            cli.close()
            if time.time() > deadline:
                raise TimeoutError("nvls: rank 0 did not publish its descriptor")
            time.sleep(0.05)
    with cli:
        _, fds, _, _ = socket.recv_fds(cli, 1, 1)
        cli.sendall(b"A")
    return fds[0]


def init_nvls(net, rank: int, world: int, tag: str = "job", group=None) -> None:
    """Bind ``net``'s arena to one NVSwitch multicast object shared by the
    ``world`` ranks (csrc/nvls.cuh): rank 0 creates it and exports a POSIX fd,
    the fd travels over a Unix socket, every rank adds its GPU, then -- after a
    barrier -- binds and maps.  torch.distributed only supplies the barriers."""
    import os
    import torch.distributed as dist
    fd = net.nvls_create(world, export=world > 1) if rank == 0 else -1
    if world > 1:
        fd = exchange_fd(fd, rank, world, tag)
    net.nvls_attach(rank, world, fd)
    if world > 1:
        dist.barrier(group=group)
    net.nvls_bind()
    if world > 1:
        dist.barrier(group=group)
        os.close(fd)


class DataParallelTrainer:
    """Mini-batch SGD/momentum over a device-resident dataset, sharded by rank."""

    def __init__(self, net, eta, mu: float, global_batch: int, rank: int = 0, world: int = 1):
        if global_batch % world != 0:
            # unequal shards would weight ranks differently under a single
            # 1/B_global scale applied per rank-local B
            raise ValueError("global batch must be divisible by the number of ranks")
        self.net, self.eta, self.mu = net, eta, mu
        self.shard = shard_batch(global_batch, rank, world)
        if net.max_batch < self.shard.rows:
            raise ValueError("network max_batch smaller than the per-rank shard")

    def step(self, X_dev: int, T_dev: int, batch_index: int, input_width: int, classes: int,
             loss_dev: int = 0) -> None:
        """One global step on rows [batch_index*B_global, ...) of the resident
        dataset; this rank processes its shard."""
        s = self.shard
        row0 = batch_index * s.rows * s.world + s.begin
        self.net.minibatch_step(X_dev + 4 * row0 * input_width, T_dev + 4 * row0 * classes, s.rows,
                                self.eta, self.mu, loss_dev)
