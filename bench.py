#!/usr/bin/env python
"""Benchmark of the B200 FC-backprop hot path (contract: see README/DESIGN).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5|c3|c2|c1|c4-<H>]

Default workload = BASELINE.json configs[4], the config the metric's
1/2/4/8-GPU numbers are quoted on: the deep MLP 4096-[4096 x 8]-10, mini-batch
4096 (global), SGD.  One "step" = one global batch through forward, dgrad,
wgrad (tcgen05 3xTF32 GEMMs) and the update; at N > 1 every rank steps its
4096/N shard and the gradient sums are all-reduced over NCCL (strong scaling:
the global batch is fixed).  Inputs: synthetic features U[0,1) and one-hot
labels from SeededRng(9) exactly like proj/tests/test_support.hpp; weights
from build_network(seed 42).

value  = samples/s with the inputs resident in HBM (device-timed, CUDA events
         on the library's stream, max over ranks, a 256 MB L2 flush between
         timed steps).
e2e    = samples/s through the public API (lane.train_minibatch over pinned
         host arrays: every step's rows are gathered into a page-locked slot,
         copied H2D on a copy stream overlapping the previous steps, and every
         step's loss is read back D2H).
--gpus N without torchrun re-launches itself under torch.distributed.run
with N ranks (and fails if fewer than N GPUs are visible); under torchrun
WORLD_SIZE must equal N.  Batch-1 online SGD (c1, c2, c4-*) has a strict
sample-to-sample dependency, so N > 1 runs N independent replicas there.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "backprop training samples/sec"
WORKLOADS = {
    # name: (input, hidden, classes, eta, epoch samples, description)
    "c1": (4, [8], 3, 0.01, 135, "4-8-3 tanh/softmax, online SGD (B=1), Iris-shaped synthetic"),
    "c2": (784, [128], 10, 0.01, 60000, "784-128-10 MNIST-shaped MLP, online SGD (B=1)"),
}
for _h in (256, 512, 1024, 2048, 4096, 8192, 16384, 100000):
    WORKLOADS[f"c4-{_h}"] = (340, [_h], 10, 1e-4, 10000 if _h <= 16384 else 1000,
                             f"340-{_h}-10 width sweep, online SGD (B=1)")
# mini-batch extension: name -> (input, hidden, classes, eta,
# global batch, momentum, batches resident, description)
MINIBATCH = {
    "c3": (1024, [4096, 4096], 10, 0.01, 256, 0.9, 16,
           "1024-4096-4096-10 wide MLP, mini-batch 256, momentum 0.9"),
    "c5": (4096, [4096] * 8, 10, 1e-3, 4096, 0.0, 4,
           "4096-[4096x8]-10 deep MLP, mini-batch 4096 (data-parallel over ranks)"),
}


def load_traffic(wl):
    """DRAM bytes per launch of the workload's dominant kernel from the
    committed ncu capture (profiles/traffic.json, tools/ncu_traffic.py)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None, None
    d = json.load(open(path)).get(wl)
    return (d["traffic_bytes_per_launch"], d["source"]) if d else (None, None)


def chain_latency(wl, plan, kernel_ms, n, clk):
    """The batch-1 window kernel's latency roofline: cycles per sample of the
    step (kernel time x the SM clock sampled under load) against the measured
    dependency floor of the per-sample chain (profiles/chain_floor.json,
    tools/ubench_chain.cu: k_chain_floor for C2's one-warp chain,
    k_chain_floor_cl for the C4 window plans' multi-warp / cluster chains)."""
    path = os.path.join(ROOT, "profiles", "chain_floor.json")
    if not plan.startswith("window") or not os.path.exists(path):
        return None
    d = json.load(open(path)).get(wl)
    if not d:
        return None
    mhz = clk.summary().get("sm_mhz") or 0
    if not mhz:
        return None
    cyc = kernel_ms / 1e3 / n * mhz * 1e6
    return {"bound": "latency", "unit": "cycles/sample", "achieved": cyc,
            "floor": d["floor_cycles_per_sample"], "frac": d["floor_cycles_per_sample"] / cyc,
            "source": d["source"], "what": d["what"]}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def cpu_reference(F, H, C, eta, X, T, samples, warmup, parallel):
    """The UNMODIFIED reference library (oracle/_ref) -- its measure() loop:
    net.forward + BackwardPlan::run per sample -- or, where it was not built,
    the plain-C restatement of the same algorithm.  Returns samples/s, kind,
    cores."""
    from oracle import pyoracle as po
    cores = os.cpu_count() or 1
    if po.ref_available():
        net = po.RefNet(F, H, C, seed=42)
        secs, _ = net.sgd_bench(X, T, warmup, samples, eta, parallel=parallel,
                                workers=cores if parallel else 1)
        return samples / secs, "reference", (cores if parallel else 1)
    net = po.OracleNet(F, H, C, seed=42)
    net.sgd_run(X, T, warmup, eta)
    t0 = time.perf_counter()
    net.sgd_run(X, T, samples, eta)
    return samples / (time.perf_counter() - t0), "port", 1


def run_reference_arm(args, wl):
    """The reference's own CPU implementation of the path (oracle/_ref: its
    proj/src/*.cpp, Release flags) on every host core (ParallelHost), timed
    with its measure() protocol (proj/src/bench.cpp:55-73: forward +
    BackwardPlan::run per sample).  Rank 0 only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as po
    cores = os.cpu_count() or 1
    if wl in MINIBATCH:
        # the reference has no mini-batch mode: its per-sample online SGD on the
        # same network, one sample per step (seconds each on the host cores);
        # the network is built once and warmed with one sample (a CPU path
        # has no state to warm beyond the first pass over the weights)
        F, H, C, eta, BG, mu, _, desc = MINIBATCH[wl]
        X, T = po.synthetic_dataset(F, C, 4, 9)
        per_step = 1
        config = {"workload": wl, "description": desc, "layers": [F] + H + [C], "global_batch": BG,
                  "momentum": mu, "eta": eta, "samples_per_step": per_step,
                  "mode": "per-sample online SGD (the reference has no mini-batch mode)"}
        if po.ref_available():
            net, kind = po.RefNet(F, H, C, seed=42), "reference"
            net.sgd_bench(X, T, 0, 1, eta, parallel=True, workers=cores)  # warm-up sample
            rates = [1.0 / net.sgd_bench(X, T, 0, 1, eta, parallel=True, workers=cores)[0]
                     for _ in range(args.steps)]
        else:
            net, kind, cores = po.OracleNet(F, H, C, seed=42), "port", 1
            net.sgd_run(X, T, 1, eta)
            rates = []
            for _ in range(args.steps):
                t0 = time.perf_counter()
                net.sgd_run(X, T, 1, eta)
                rates.append(1.0 / (time.perf_counter() - t0))
    else:
        F, H, C, eta, n_epoch, desc = WORKLOADS[wl]
        X, T = po.synthetic_dataset(F, C, min(n_epoch, 4096), 9)
        per_ms = {"c1": 0.003, "c2": 1.0}.get(wl, 0.6 * (F * H[0] + H[0] * C) / 1e5)
        per_step = max(10, int(4000.0 / per_ms / max(1, args.steps + args.warmup)))  # ~4 s of CPU
        per_step = min(per_step, 100000)
        config = {"workload": wl, "description": desc, "layers": [F] + H + [C], "batch": 1,
                  "samples_per_step": per_step, "eta": eta}
        rates = []
        kind = "port"
        for s in range(args.warmup + args.steps):
            r, kind, cores = cpu_reference(F, H, C, eta, X, T, per_step, 2, parallel=True)
            if s >= args.warmup:
                rates.append(r)
    value = float(np.mean(rates))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * per_step / value, "higher_is_better": True,
            "scaling": "strong" if wl in MINIBATCH else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config,
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                             "sample": f"{per_step} online-SGD sample(s) per step through the "
                                       f"reference's forward + BackwardPlan::run on ParallelHost "
                                       f"({cores} workers)"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def dominant_gemm(dev, widths, rows, stream):
    """fp32-equivalent TFLOP/s of the tensor-core GEMMs alone over the step's
    GEMM shapes (same kernels, precision scheme and shapes as inside the
    captured step graph, which cannot be timed per kernel: lane_b200_gemm with
    use_tc = 5, the step's own choice), and their share of the step's flops."""
    import ctypes as C
    import torch
    from paper_2001_04206_b200 import _native
    L = _native.lib()
    shapes = []  # (op, M, N, K): op 0 NN (fwd), 1 NT (dgrad), 2 TN (wgrad)
    for l, (i, o) in enumerate(zip(widths[:-1], widths[1:])):
        if o < 64:
            continue  # the 10-wide output layer runs on SIMT kernels
        shapes.append((0, rows, o, i))
        shapes.append((2, i, o, rows))
        if l > 0:
            shapes.append((1, rows, i, o))
    tot_f, tot_ms = 0.0, 0.0
    for op, M, N, K in shapes:
        a = torch.randn(M * K, device="cuda")
        b = torch.randn(N * K, device="cuda")
        c = torch.empty(M * N, device="cuda")
        # the 3xF16 operand maxima once per shape, outside the timed calls, as
        # the step computes them once per step (rows of op(A), columns of op(B))
        ar, br = (K, M) if op == 2 else (M, K), (N, K) if op == 1 else (K, N)
        amx = [torch.empty(ar[0], dtype=torch.int32, device="cuda"), torch.empty(ar[1], dtype=torch.int32, device="cuda")]
        bmx = [torch.empty(br[0], dtype=torch.int32, device="cuda"), torch.empty(br[1], dtype=torch.int32, device="cuda")]
        for t, (r_, c_), mx in ((a, ar, amx), (b, br, bmx)):
            assert L.lane_b200_absmax(dev._p, C.c_void_p(t.data_ptr()), r_, c_, C.c_void_p(mx[0].data_ptr()),
                                      C.c_void_p(mx[1].data_ptr())) == 0, L.lane_b200_last_error()
        amax = amx[1] if op == 2 else amx[0]
        bmax = bmx[0] if op == 1 else bmx[1]
        def call():
            rc = L.lane_b200_gemm_ex(dev._p, op, M, N, K, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                     C.c_void_p(c.data_ptr()), None, None, None, 0, 5,
                                     C.c_void_p(amax.data_ptr()), C.c_void_p(bmax.data_ptr()))
            assert rc == 0, L.lane_b200_last_error()
        for _ in range(2):
            call()
        dev.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            call()
        e1.record(stream)
        e1.synchronize()
        tot_ms += e0.elapsed_time(e1) / 10
        tot_f += 2.0 * M * N * K
        del a, b, c
    P = sum(i * o for i, o in zip(widths[:-1], widths[1:]))
    step_f = (6 * P - 2 * widths[0] * widths[1]) * rows
    return (tot_f / (tot_ms / 1e3) / 1e12 if tot_ms else None), tot_f / step_f


def uses_h3(widths, rows):
    """True when the step's tensor-core GEMMs run the 3xF16 kernel (gemm.cuh
    tc_use_h3: tall CTA-pair shapes with K >= 2048), unless overridden."""
    mode = os.environ.get("LANE_B200_TC_PREC", "auto")
    if mode in ("f16", "tf32"):
        return mode == "f16"
    big = [(rows, o, i) for i, o in zip(widths[:-1], widths[1:]) if o >= 64]
    return bool(big) and all((M >= 1024 or (M >= 512 and K >= 2048)) and K >= 2048 and N >= 256
                             for M, N, K in big)


def measure_tf32_peak(dtype: str = "tf32") -> float:
    """Dense tensor-core TFLOP/s of this GPU as cuBLAS reaches it at 8192^3,
    best of 10 (CUDA events): fp32 matmul with TF32 enabled ("tf32"), or a
    plain fp16 matmul ("f16")."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        dt = torch.float16 if dtype == "f16" else torch.float32
        a = torch.randn(n, n, device="cuda", dtype=dt)
        b = torch.randn(n, n, device="cuda", dtype=dt)
        c = torch.empty(n, n, device="cuda", dtype=dt)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return 2.0 * n ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def run_minibatch(args, wl):
    """Mini-batch workloads (C3, C5): one step = one global batch through
    forward, dgrad, wgrad (tcgen05 3xTF32 GEMMs) and the SGD/momentum update;
    at N>1 each rank steps its shard and the library all-reduces the gradient
    sums once per step over NCCL."""
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from oracle import pyoracle as po  # synthetic data generator + cpu_baseline only
    from paper_2001_04206_b200 import lane, parallel

    F, H, C, eta, BG, mu, nb, desc = MINIBATCH[wl]
    dev = lane.Device(local)
    if world > 1:
        parallel.init_comm(dev, rank, world)
    rows = BG // world
    net = lane.build_network(F, H, C, seed=42, device=dev, max_batch=rows)
    if world > 1 and args.exchange == "nvls":
        parallel.init_nvls(net, rank, world, tag=os.environ.get("MASTER_PORT", "bench"))
    trainer = parallel.DataParallelTrainer(net, eta, mu, BG, rank, world)
    X, T = po.synthetic_dataset(F, C, nb * BG, 9)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
    stream = torch.cuda.ExternalStream(dev.stream, device=torch.device("cuda", local))
    for s in range(args.warmup):
        trainer.step(xd, td, s % nb, F, C)
    dev.sync()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = dev.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (outside the events)
            evs[s][0].record(stream)
            trainer.step(xd, td, s % nb, F, C)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    launches = dev.kernel_launches - launches0
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = BG * args.steps / (ms / 1000.0)

    # e2e: through the public trainer (lane.train_minibatch) over pinned host
    # arrays: every step's rows are gathered into a page-locked slot and copied
    # H2D on the library's copy stream (overlapping the previous steps), and
    # every step's loss is read back D2H (async, 8 bytes)
    Xh = torch.from_numpy(X).pin_memory().numpy()
    Th = torch.from_numpy(T).pin_memory().numpy()
    ds = lane.DataSet(Xh, Th)
    # at least 20 steps, so the first step's exposed H2D and the final sync
    # stay a small share of the timed call
    epochs = max(1, -(-max(20, min(args.steps, 40)) // nb))
    lane.train_minibatch(net, ds, rows, eta, mu, epochs=1, shuffle=False)  # warm: staging + graph
    e2e_steps = epochs * nb
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lane.train_minibatch(net, ds, rows, eta, mu, epochs=epochs, shuffle=False)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = BG * e2e_steps / e2e_s

    widths = [F] + H + [C]
    P = sum(a * b for a, b in zip(widths[:-1], widths[1:]))
    P0 = widths[0] * widths[1]
    flops = (6 * P - 2 * P0) * BG  # fwd 2P + wgrad 2P + dgrad 2(P - P0) per sample
    step_tf = flops / (ms / args.steps / 1000.0) / 1e12
    gemm_tf, gemm_share = dominant_gemm(dev, widths, rows, stream)
    # the denominator: this box's dense tensor rate for the MMA kind the step
    # runs (cuBLAS at 8192^3, best of 10: fp16 for the 3xF16 kernel, fp32 with
    # TF32 for the 3xTF32 kernels), / 3 for the 3 MMAs per fp32 product
    h3 = uses_h3(widths, rows)
    tc_rate = measure_tf32_peak("f16" if h3 else "tf32")
    peak = tc_rate / 3.0
    nominal = 2250.0 / (1.0 if h3 else 2.0) / 3.0  # NVIDIA's dense fp16 2.25 PF/s (TF32: half)
    kernel = "k_gemm_h3" if h3 else "k_gemm_tc"
    gemm_desc = ("tcgen05 kind::f16, 3xF16 (power-of-two row/column scales; fp32-accurate, 1e-5 "
                 "condition-aware)" if h3 else "tcgen05 kind::tf32, 3xTF32 (fp32-accurate, 1e-5 condition-aware)")
    # the step's two sequential phases each have a floor: the GEMMs on the tensor
    # pipe and the update streaming W, V and G (read + write, 24 B/param) from
    # HBM; the next step's forward needs the updated weights, so they add
    hbm_peak, _ = load_peaks()
    n_param = sum(a * b + b for a, b in zip(widths[:-1], widths[1:]))
    floor_tensor_us = flops * gemm_share / (peak * 1e12) * 1e6
    floor_update_us = (24.0 if mu else 20.0) * n_param / (hbm_peak * 1e9) * 1e6
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl, "description": desc, "layers": widths, "global_batch": BG,
                       "rows_per_rank": rows, "momentum": mu, "eta": eta, "parallelism": f"dp{world}",
                       "exchange": (args.exchange if world > 1 else "none"),
                       "gemm": gemm_desc,
                       "l2": "256 MB buffer written between timed steps"},
            "roofline": {"bound": "tensor", "kernel": kernel, "achieved": gemm_tf, "peak": peak,
                         "unit": "TFLOP/s", "frac": gemm_tf / peak if gemm_tf else None,
                         "traffic": load_traffic(wl)[0], "traffic_source": load_traffic(wl)[1],
                         "how": "the step's tensor-core GEMM shapes (fwd/dgrad/wgrad of the 4096-wide "
                                "layers) replayed through lane_b200_gemm_ex (the step's kernel choice; "
                                "3xF16 operand maxima computed once per shape outside the timing, as "
                                "the step computes them once per step), CUDA events on the library "
                                "stream, 10 reps each; algorithmic flops 2MNK per launch",
                         "peak_kind": f"measured: cuBLAS dense {'fp16' if h3 else 'TF32'} 8192^3 on this "
                                      f"GPU ({tc_rate:.0f} TF/s) / 3 (MMAs per fp32 product)",
                         "frac_of_nominal": gemm_tf / nominal if gemm_tf else None,
                         "flop_share_of_step": gemm_share,
                         "step": {"achieved": step_tf, "frac": step_tf / peak,
                                  "scope": "whole step (every kernel incl. the HBM-bound update) / "
                                           "step time"},
                         "step_floor": {"tensor_us": floor_tensor_us, "hbm_update_us": floor_update_us,
                                        "frac": (floor_tensor_us + floor_update_us) / (ms / args.steps * 1e3),
                                        "how": "GEMM flops at the measured 3-MMA peak + the update's "
                                               "20 (SGD) / 24 (momentum) B/param at the measured HBM "
                                               "peak, against the measured step time"},
                         "algorithmic_flops_per_step": flops},
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": rows * (F + C) * 4,
                    "d2h_bytes_per_step": 8},
            "gpu_launches": int(launches), "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu:
        v, kind, cores = cpu_reference(F, H, C, eta, X[:4], T[:4], 1, 0, parallel=True)
        line["cpu_baseline"] = {"value": v, "unit": "samples/s", "cores": cores, "kind": kind,
                                "sample": "1 sample of per-sample online SGD through the reference "
                                          "(it has no mini-batch mode), ParallelHost"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_paper_table(args):
    """The paper's per-kernel table (340-100000-10):
    the reference's own lane-bench (lane::run_benchmark through oracle/_ref,
    serial and parallel on every host core) and the B200 lane-bench CLI
    (paper_2001_04206_b200/lib/lane-bench) on the same synthetic dataset,
    merged into one report (speedup = reference serial mean / device mean)."""
    import ctypes as C
    import tempfile
    from oracle import pyoracle as po  # CPU reference leg + data generator only
    from paper_2001_04206_b200 import _build, lane

    F, Cn, H = 340, 10, args.fc_neurons
    X, T = po.synthetic_dataset(F, Cn, 64, 9)
    tmp = tempfile.mkdtemp()
    data = os.path.join(tmp, "paper_340x10.csv")
    lane.save_dataset(lane.DataSet(X, T), data)
    warm, iters = max(1, args.warmup), max(1, args.steps)
    ref_csv = os.path.join(tmp, "ref.csv")
    if po.ref_available():
        f = po.ref_lib().lr_run_benchmark
        f.restype = C.c_long
        f.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float, C.c_size_t, C.c_size_t,
                      C.c_size_t, C.c_int, C.c_uint, C.c_uint64, C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64)]
        buf, h = C.create_string_buffer(1 << 14), C.c_uint64()
        if f(data.encode(), F, Cn, H, 1e-4, warm, iters, 1, 1, os.cpu_count() or 1, 42, buf, 1 << 14,
             C.byref(h)) < 0:
            raise RuntimeError(po.ref_lib().lr_last_error().decode())
        open(ref_csv, "w").write(buf.value.decode())
    _build.build()
    cmd = [_build.CLI, "--dataset", data, "--features", str(F), "--classes", str(Cn), "--fc-neurons", str(H),
           "--eta", "1e-4", "--warmup", str(max(warm, 20)), "--iters", str(max(iters, 20)), "--format", "md"]
    if os.path.exists(ref_csv):
        cmd += ["--baseline-csv", ref_csv]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True)
    print(f"lane-bench {F}-{H}-{Cn}, eta 1e-4; reference: warmup {warm}, iters {iters}, "
          f"{os.cpu_count()} host threads; b200: warmup {max(warm, 20)}, iters {max(iters, 20)}")
    print(out.stdout, end="", flush=True)


def self_launch(args) -> int:
    """--gpus N outside torchrun: N ranks under torch.distributed.run on this
    node (127.0.0.1 rendezvous).  Refuses loudly when fewer than N GPUs are
    visible instead of silently running one rank."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS) + sorted(MINIBATCH))
    ap.add_argument("--epoch", type=int, default=0, help="override samples per step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "nvls"],
                    help="mini-batch gradient exchange at N > 1: per-layer NCCL allreduces (default) or the "
                         "NVLS fused switch-reduce + update (csrc/nvls.cuh; needs a fabric-attached node)")
    ap.add_argument("--paper-table", action="store_true",
                    help="the paper's per-kernel lane-bench table (reference serial/parallel + b200)")
    ap.add_argument("--fc-neurons", type=int, default=100000, help="--paper-table hidden width")
    args = ap.parse_args()
    wl = args.workload
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and not args.paper_table:
        sys.exit(self_launch(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}")
    if args.paper_table:
        run_paper_table(args)
        return
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return
    if wl in MINIBATCH:
        run_minibatch(args, wl)
        return

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from oracle import pyoracle as po  # synthetic data generator + cpu_baseline only
    from paper_2001_04206_b200 import lane

    F, H, C, eta, n, desc = WORKLOADS[wl]
    if args.epoch:
        n = args.epoch
    dev = lane.Device(local)
    X, T = po.synthetic_dataset(F, C, n, 9)
    net = lane.build_network(F, H, C, seed=42, device=dev)
    xd, td = dev.alloc(X.nbytes), dev.alloc(T.nbytes)
    dev.h2d(xd, X)
    dev.h2d(td, T)
    dev.sync()

    stream = torch.cuda.ExternalStream(dev.stream, device=torch.device("cuda", local))
    for _ in range(args.warmup):
        net.sgd_stream(xd, td, n, n, eta)
    dev.sync()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize()
    launches0 = dev.kernel_launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for s in range(args.steps):
            kev[s][0].record(stream)
            net.sgd_stream(xd, td, n, n, eta)
            kev[s][1].record(stream)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = dev.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1)
    step_ms = [a.elapsed_time(b) for a, b in kev]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * n * args.steps / (ms / 1000.0)

    # ---- end to end through the public API: lane.train over pinned host arrays ----
    Xh = torch.from_numpy(X).pin_memory().numpy()
    Th = torch.from_numpy(T).pin_memory().numpy()
    ds = lane.DataSet(Xh, Th)
    # one train() call over several epochs (a step = one epoch), as a user
    # trains: max_error 0, so it stops early only on an exactly zero loss
    lane.train(net, ds, lane.TrainerConfig(lane.LearningRate(eta), 0.0, 2, 42))  # warm
    cfg = lane.TrainerConfig(lane.LearningRate(eta), 0.0, max(1, min(args.steps, 10)), 42)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = len(lane.train(net, ds, cfg))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = world * n * e2e_steps / e2e_s

    # ---- roofline of the dominant kernel (the fused online-SGD plan) ----
    plan = net.sgd_plan()
    peak, peak_kind = load_peaks()
    P = sum(a * b + b for a, b in zip([F] + H, H + [C]))
    # per sample 4P (forward read of W) + 8P (update read+write
    # of W) + 12 B per activation of every width (x, z, a / delta)
    bytes_per_sample = 12 * P + 12 * (F + sum(H) + C)
    kernel_ms = float(np.mean(step_ms))
    achieved = bytes_per_sample * n / (kernel_ms / 1000.0) / 1e9

    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl, "description": desc, "layers": [F] + H + [C], "batch": 1,
                       "samples_per_step": n, "eta": eta, "numerics": "fast",
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": f"inputs {X.nbytes + T.nbytes} B > 126 MB L2, streamed each step"
                       if X.nbytes + T.nbytes > 126e6 else "inputs fit in L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(wl)[0],
                         "traffic_source": load_traffic(wl)[1],
                         "peak_kind": peak_kind,
                         "kernel": {"window": "k_sgd_window", "cluster": "k_sgd_cluster",
                                    "grid": "k_sgd_grid"}.get(plan.split()[0], "layer kernels"),
                         "plan": plan,
                         "algorithmic_bytes_per_sample": bytes_per_sample,
                         "note": "algorithmic bytes per sample = SURVEY 8(d): 12 B/param (forward "
                                 "read + update read/write of W) + 12 B/activation, the HBM floor of "
                                 "a design that streams the weights; this kernel keeps them on chip "
                                 "(DRAM traffic is the inputs only) and is bound by the serial "
                                 "per-sample chain (DESIGN.md section 4.1); achieved uses the whole "
                                 "step (Gram pre-pass + kernel + G/DW), CUDA events on the library "
                                 "stream",
                         "latency": chain_latency(wl, plan, kernel_ms, n, clk)},
            "e2e": {"value": e2e, "unit": "samples/s",
                    "h2d_bytes_per_step": int(X.nbytes + T.nbytes),
                    "d2h_bytes_per_step": 8 * 2 + 4},  # EpochStats (loss sum, hits) + the device error flag
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu:
        Xs, Ts = X[:2000], T[:2000]
        per_ms = {"c1": 0.003, "c2": 1.0}.get(wl, 0.6 * P / 1e5)
        samples = int(max(20, min(20000, 8000.0 / per_ms)))  # ~8 s of single-core CPU
        v, kind, cores = cpu_reference(F, H, C, eta, Xs, Ts, samples, 5, parallel=False)
        line["cpu_baseline"] = {"value": v, "unit": "samples/s", "cores": cores, "kind": kind,
                                "sample": f"{samples} online-SGD samples of the same workload "
                                          f"(reference forward + BackwardPlan::run, SerialHost)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for p in (xd, td):
        dev.free(p)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
