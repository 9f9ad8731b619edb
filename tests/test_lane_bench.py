"""lane-bench for the B200 path (paper_2001_04206_b200/csrc/lane_bench.cpp):
the reference's CLI flags and report format (proj/tools/lane_bench.cpp,
proj/src/bench.cpp), a "b200" device row per kernel, and -- in strict
numerics -- the reference's final weights hash (tests/golden/lane_bench.json,
made by tests/golden/make_lane_bench_golden.py from the unmodified
reference)."""
import json
import math
import os
import subprocess

import pytest

from paper_2001_04206_b200 import _build

HERE = os.path.dirname(os.path.abspath(__file__))
IRIS = os.path.join(HERE, "golden", "iris_normalized.txt")
GOLD = json.load(open(os.path.join(HERE, "golden", "lane_bench.json")))


def cli():
    _build.build()
    return _build.CLI


def run(*args, timeout=300):
    return subprocess.run([cli(), *map(str, args)], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("args,msg", [
    ((), "--dataset is required"),
    (("--dataset", IRIS, "--device", "serial"), "--device must be 'b200'"),
    (("--dataset", IRIS, "--format", "xml"), "--format must be 'csv' or 'md'"),
    (("--dataset", IRIS, "--iters", "0"), "timed_iters must be >= 1"),
    (("--dataset", IRIS, "--classes", "1"), "invalid network topology"),
    (("--dataset", IRIS, "--eta", "0"), "eta must be positive"),
    (("--dataset", IRIS, "--fc-neurons", "abc"), "bad value"),
    (("--dataset", IRIS, "--warmup", "-1"), "bad value"),
    (("--dataset", IRIS, "--bogus"), "unknown option"),
])
def test_cli_configuration_errors_exit_2(args, msg):
    # lane_bench.cpp:53-69: configuration errors -> exit 2 (no GPU touched)
    out = run(*args)
    assert out.returncode == 2 and msg in out.stderr, out.stderr


def test_cli_help():
    out = run("--help")
    assert out.returncode == 0 and "--fc-neurons" in out.stdout and "--baseline-csv" in out.stdout


def parse_csv(text):
    lines = text.strip().splitlines()
    assert lines[0] == "kernel,device,mean_ms,copy_in_ms,kernel_ms,copy_out_ms,speedup"
    rows = [ln.split(",") for ln in lines[1:]]
    for r in rows:
        assert len(r) == 7
        for v in r[2:]:
            assert v == "nan" or len(v.split(".")[1]) == 3  # "%.3f" (bench.cpp:193-196)
    return rows


@pytest.mark.gpu
@pytest.mark.parametrize("g", GOLD, ids=lambda g: f"fc{g['fc_neurons']}-e{g['enlarge']}-s{g['seed']}")
def test_strict_final_weights_hash_matches_reference(g):
    out = run("--dataset", IRIS, "--features", 4, "--classes", 3, "--fc-neurons", g["fc_neurons"],
              "--eta", g["eta"], "--warmup", g["warmup"], "--iters", g["iters"], "--enlarge", g["enlarge"],
              "--seed", g["seed"], "--numerics", "strict", "--print-hash")
    assert out.returncode == 0, out.stderr
    assert f"final_weights_hash={g['final_weights_hash']}" in out.stderr
    rows = parse_csv(out.stdout)
    assert [r[:2] for r in rows] == [["softmax_backward", "b200"], ["fc_backward", "b200"]]
    for r in rows:
        mean, cin, k, cout = map(float, r[2:6])
        assert k > 0 and cout == 0 and abs(mean - (cin + k + cout)) <= 0.0015
        assert math.isnan(float(r[6]))  # no baseline -> no speedup


@pytest.mark.gpu
def test_baseline_merge_and_md(tmp_path):
    base = tmp_path / "ref.csv"
    base.write_text("kernel,device,mean_ms,copy_in_ms,kernel_ms,copy_out_ms,speedup\n"
                    "softmax_backward,serial,0.500,0.100,0.300,0.100,1.000\n"
                    "softmax_backward,parallel,0.400,0.100,0.200,0.100,1.250\n"
                    "fc_backward,serial,8.000,1.000,6.000,1.000,1.000\n"
                    "fc_backward,parallel,2.000,0.500,1.000,0.500,4.000\n")
    out = run("--dataset", IRIS, "--warmup", 20, "--iters", 10, "--baseline-csv", base)
    assert out.returncode == 0, out.stderr
    rows = parse_csv(out.stdout)
    assert [r[:2] for r in rows] == [["softmax_backward", "serial"], ["softmax_backward", "parallel"],
                                     ["softmax_backward", "b200"], ["fc_backward", "serial"],
                                     ["fc_backward", "parallel"], ["fc_backward", "b200"]]
    for r, serial in ((rows[2], 0.5), (rows[5], 8.0)):
        mean = float(r[2])  # printed at 3 decimals; the speedup uses the unrounded mean
        assert serial / (mean + 0.0005) - 1e-3 <= float(r[6]) <= serial / max(mean - 0.0005, 1e-9) + 1e-3
    md = tmp_path / "out.md"
    out = run("--dataset", IRIS, "--warmup", 5, "--iters", 3, "--format", "md", "--out", md)
    assert out.returncode == 0 and out.stdout == ""
    text = md.read_text().splitlines()
    assert text[0] == "| kernel | device | mean_ms | copy_in_ms | kernel_ms | copy_out_ms | speedup |"
    assert text[1] == "|---|---|---|---|---|---|---|" and len(text) == 4
