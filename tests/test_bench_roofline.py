"""bench.py's latency roofline (no GPU): the measured chain floors in
profiles/chain_floor.json are looked up per workload, only for the window
plans, and turned into cycles per sample with the sampled SM clock."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class _Clk:
    def __init__(self, mhz):
        self.mhz = mhz

    def summary(self):
        return {"sm_mhz": self.mhz}


def test_chain_floor_file_covers_window_workloads():
    d = json.load(open(os.path.join(ROOT, "profiles", "chain_floor.json")))
    for wl in ("c2", "c4-256", "c4-512", "c4-1024", "c4-2048", "c4-4096", "c4-8192"):
        assert wl in d, wl
        assert d[wl]["floor_cycles_per_sample"] > 0
        assert d[wl]["source"] and d[wl]["what"]


@pytest.mark.parametrize("wl", ["c2", "c4-4096"])
def test_chain_latency_cycles(wl):
    floor = json.load(open(os.path.join(ROOT, "profiles", "chain_floor.json")))[wl]["floor_cycles_per_sample"]
    # 10,000 samples in 5 ms at 2000 MHz = 1000 cycles per sample
    r = bench.chain_latency(wl, "window 1x1", 5.0, 10000, _Clk(2000.0))
    assert r["bound"] == "latency" and r["unit"] == "cycles/sample"
    assert r["achieved"] == pytest.approx(1000.0)
    assert r["frac"] == pytest.approx(floor / 1000.0)


def test_chain_latency_only_for_window_plans():
    assert bench.chain_latency("c2", "grid", 5.0, 10000, _Clk(2000.0)) is None
    assert bench.chain_latency("c4-16384", "window", 5.0, 10000, _Clk(2000.0)) is None  # no floor measured
    assert bench.chain_latency("c2", "window", 5.0, 10000, _Clk(0)) is None  # no clock sample


def test_gpus_n_refuses_without_n_gpus(tmp_path):
    # --gpus N outside torchrun self-launches N ranks, or fails loudly: it never
    # silently runs one rank (this container has no GPU)
    import subprocess
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs to launch")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "needs 2 visible GPUs" in r.stderr
    assert r.stdout.strip() == ""  # no bench line
