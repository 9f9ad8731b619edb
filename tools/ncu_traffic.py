"""DRAM traffic per launch of each workload's dominant kernel, from ncu, into
profiles/traffic.json (bench.py reports it as roofline.traffic).

    python tools/ncu_traffic.py            # on the GPU box (runs ncu)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = {  # workload: (bench args, kernel-name substring)
    "c2": (["--workload", "c2"], "k_sgd_window"),
    "c3": (["--workload", "c3"], "k_gemm_tc"),
    "c5": (["--workload", "c5"], "k_gemm_h3"),
    # (the cluster window plans, H = 512..8192, fail to launch under ncu's
    # replay -- LaunchFailed -- so the non-cluster H = 256 plan stands in)
    "c4-256": (["--workload", "c4-256"], "k_sgd_window"),
    "c4-16384": (["--workload", "c4-16384"], "k_sgd_grid"),
}


def main():
    only = sys.argv[1:]
    path = os.path.join(ROOT, "gpurun_out", "traffic.json")
    out = json.load(open(path)) if only and os.path.exists(path) else {}
    for wl, (args, kname) in RUNS.items():
        if only and wl not in only:
            continue
        log = os.path.join(ROOT, "gpurun_out", f"traffic_{wl}.csv")
        cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
               "--clock-control", "none", "-k", f"regex:{kname}", "--csv", "--log-file", log,
               sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu", *args]
        subprocess.run(cmd, cwd=ROOT, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=1200)
        rows = [r for r in csv.reader(open(log)) if len(r) > 5]
        h = rows[0]
        ii, mi, vi, ki = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name")
        per = {}
        for r in rows[1:]:
            d = per.setdefault(r[ii], {"kernel": r[ki]})
            d[r[mi]] = float(r[vi].replace(",", ""))
        launches = list(per.values())
        if wl == "c2" or wl.startswith("c4"):
            # the bench's 60,000-sample launches (the e2e leg streams smaller chunks)
            tmax = max(l["gpu__time_duration.sum"] for l in launches)
            launches = [l for l in launches if l["gpu__time_duration.sum"] >= 0.9 * tmax]
        # mini-batch: the mean over the step's GEMM launches (all shapes)
        if not launches:
            print(wl, "no launches captured", flush=True)
            continue
        rd = sum(l["dram__bytes_read.sum"] for l in launches) / len(launches)
        wr = sum(l["dram__bytes_write.sum"] for l in launches) / len(launches)
        out[wl] = {"kernel": kname, "launches_captured": len(launches), "dram_read_bytes": rd,
                   "dram_write_bytes": wr, "traffic_bytes_per_launch": rd + wr,
                   "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:{kname} "
                             f"python bench.py --steps 1 --warmup 3 {' '.join(args)}"}
        print(wl, json.dumps(out[wl]), flush=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
