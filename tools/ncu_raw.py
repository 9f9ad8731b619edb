"""Pick metrics out of `ncu --page raw --csv` exports (one kernel per file).

    python tools/ncu_raw.py file1.csv [file2.csv ...] [-m regex]
"""
import csv
import re
import sys

DEFAULT = (r"^(gpu__time_duration.sum|sm__cycles_elapsed.avg.per_second|dram__bytes_(read|write)\.sum|"
           r"sm__pipe_tensor.*cycles_active.avg.pct_of_peak_sustained_(active|elapsed)|"
           r"sm__throughput.avg.pct_of_peak_sustained_elapsed|launch__grid_size|"
           r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum|smsp__inst_executed.sum|"
           r"sm__warps_active.avg.pct_of_peak_sustained_active|lts__t_bytes.sum|"
           r"smsp__average_warp(s_issue_stalled|_latency_issue_stalled)_.*_per_issue_active.ratio)$")


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    vals = rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def main():
    args = sys.argv[1:]
    pat = DEFAULT
    if "-m" in args:
        i = args.index("-m")
        pat = args[i + 1]
        args = args[:i] + args[i + 2:]
    ds = [load(a) for a in args]
    keys = [k for k in ds[0] if re.search(pat, k)]
    print("| metric | " + " | ".join(a.split("/")[-1].replace("_raw.csv", "") for a in args) + " | unit |")
    print("|---|" + "---:|" * len(args) + "---|")
    for k in keys:
        vs = [d.get(k, ("", ""))[0] for d in ds]
        print(f"| `{k}` | " + " | ".join(vs) + f" | {ds[0][k][1]} |")


if __name__ == "__main__":
    main()
