"""Warp-stall summary of an `ncu --page source --csv` (SASS) export.

usage: python tools/ncu_stalls.py src.csv [top_lines]
Prints, per kernel section, the stall-reason breakdown and the hottest SASS
instructions (by warp-stall samples).
"""
import collections
import csv
import sys


def sections(path):
    rows = list(csv.reader(open(path)))
    out, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            out.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    return out


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    for sec in sections(path):
        h = sec["rows"][0]
        data = [r for r in sec["rows"][1:] if len(r) == len(h) and r[2].isdigit()]
        cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        agg = collections.Counter()
        for r in data:
            for i in cols:
                agg[h[i]] += int(r[i] or 0)
        tot = sum(agg.values()) or 1
        print(sec["name"][:70], "samples", tot)
        print("   ", [(k[6:], round(100 * v / tot, 1)) for k, v in agg.most_common(8)])
        si = h.index("Warp Stall Sampling (All Samples)")
        for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
            print("      ", r[si].rjust(6), r[1][:90])


if __name__ == "__main__":
    main()
