"""Top CUDA source lines by warp-stall samples from an ncu report.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [N] [kernel-substring]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] and len(r) > 4 and r[2] == "-":
            try:
                agg[(cur, int(r[0]))] = (int(r[4]), int(r[5]), r[1].strip()[:90])
            except ValueError:
                pass
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"total stall samples {tot}")
    for (f, ln), (a, ni, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{a:7d} {100 * a / tot:5.1f}% (not-issued {ni:6d}) {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
