"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump
per CUDA source line: share of warp-stall samples and of instructions."""
import collections
import csv
import os
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=40):
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    src = {}
    fname, line, h = "?", None, None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname, line = os.path.basename(r[1]), None
            continue
        if r[0] == "Line No":
            h = r
            i_s = h.index("Warp Stall Sampling (All Samples)")
            i_i = h.index("Instructions Executed")
            continue
        if h is None or len(r) < len(h):
            continue
        if r[0]:
            line = (fname, int(r[0]))
            src[line] = r[1]
        if line is None or not r[2]:
            continue
        agg[line][0] += num(r[i_s])
        agg[line][1] += num(r[i_i])
    ts = sum(a[0] for a in agg.values()) or 1
    ti = sum(a[1] for a in agg.values()) or 1
    print(f"samples {ts:.0f} instructions {ti:.0f}")
    for (f, ln), (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * s / ts:5.1f}%s {100 * i / ti:5.1f}%i  {f}:{ln:<5} {src.get((f, ln), '').strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
