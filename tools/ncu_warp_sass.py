"""Stall breakdown of one warp role's SASS from an ncu report (source page,
per-instruction warp-state samples).  Selects instructions by execution count.

    python tools/ncu_warp_sass.py REPORT EXEC_COUNT [TOL] [TOP]
"""
import csv
import subprocess
import sys


def main():
    rep, cnt = sys.argv[1], int(sys.argv[2])
    tol = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
    sel = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            ex = int(r[ix["Instructions Executed"]])
        except ValueError:
            continue
        if abs(ex - cnt) <= tol:
            sel.append(r)
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]]) for r in sel)
    print(f"{len(sel)} instructions executed ~{cnt} times; {tot} samples "
          f"({tot / max(1, cnt):.2f} samples per execution)")
    agg = {h: sum(int(r[ix[h]] or 0) for r in sel) for h in reasons}
    for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {h:24s} {v:8d} {100 * v / max(1, tot):5.1f}%")
    print("top instructions:")
    sel.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]]))
    for r in sel[:top]:
        why = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
        print(f"  {r[ix['Address']][-5:]} {int(r[ix['Warp Stall Sampling (All Samples)']]):6d}  "
              f"{r[ix['Source']].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main()
