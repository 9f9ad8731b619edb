"""NVLS fused gradient exchange + update (csrc/nvls.cuh).

On one GPU the NVLS state has a single member (a one-device multicast object,
or the "local" state where the driver refuses one), so the reduce returns the
rank's own sums and the step must equal the plain one-rank step bit for bit
(same update sequence as k_momentum_update_all), through the VMM arena, the
slice bounds and the in-stream barriers.  The descriptor
exchange of the multi-rank setup is tested on CPU with two processes."""
import multiprocessing as mp
import os
import tempfile

import numpy as np
import pytest

from paper_2001_04206_b200 import parallel


def _recv(tag, q):
    fd = parallel.exchange_fd(-1, 1, 2, tag, timeout=30)
    with os.fdopen(fd, "rb") as f:
        f.seek(0)
        q.put(f.read())


def test_exchange_fd_two_processes():
    tag = f"test{os.getpid()}"
    with tempfile.TemporaryFile() as f:
        f.write(b"multicast handle stand-in")
        f.flush()
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_recv, args=(tag, q))
        p.start()
        parallel.exchange_fd(f.fileno(), 0, 2, tag, timeout=30)
        got = q.get(timeout=30)
        p.join(30)
    assert p.exitcode == 0
    assert got == b"multicast handle stand-in"


@pytest.mark.gpu
@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_nvls_single_rank_step_bitwise(mu):
    from oracle import pyoracle as po  # checker-side data generator
    from paper_2001_04206_b200 import lane
    dev = lane.Device(0)
    F, H, C, B = 1024, [512, 512], 10, 64
    X, T = po.synthetic_dataset(F, C, 3 * B, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    plain = lane.build_network(F, H, C, seed=42, device=dev, max_batch=B)
    fused = lane.build_network(F, H, C, seed=42, device=dev, max_batch=B)
    fused.nvls_create(1, export=False)
    fused.nvls_attach(0, 1)
    fused.nvls_bind()
    # "multicast" on a fabric-attached GPU; "local" where the driver refuses a
    # single-member multicast object (the multimem instructions then do not run)
    assert fused.nvls_mode() in ("multicast", "local")
    assert plain.nvls_mode() == "off"
    for s in range(3):
        for net in (plain, fused):
            net.minibatch_step(xd + 4 * s * B * F, td + 4 * s * B * C, B, 0.01, mu)
    dev.sync()
    for a, b in zip(plain.hidden + [plain.output], fused.hidden + [fused.output]):
        for buf in (lane.W, lane.B, lane.G, lane.DW, lane.DELTA_BIASES, lane.BIAS_GRAD):
            np.testing.assert_array_equal(a.read(buf), b.read(buf))


@pytest.mark.gpu
def test_nvls_kernels_compiled_with_multimem():
    import subprocess
    from paper_2001_04206_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    assert "k_nvls_update" in sass
    # the multicast instantiation: multimem.ld_reduce is LDGMC (switch-reduced
    # vector load); multimem.st / .red are STG / REDG ...STRONG.SYS to the
    # multicast address
    assert "LDGMC.E.ADD.F32x4" in sass, "no multimem.ld_reduce in the SASS"
