"""Stall samples of an ncu source page (SASS), summed over instruction classes and over the hot
region (between the first and last instruction of a given opcode).
  python tools/stall_regions.py <src.csv> [HOTOPCODE]"""
import csv
import sys
from collections import defaultdict


def main(p, hot="FFMA2"):
    rows = list(csv.reader(open(p)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    R = [r for r in rows[2:] if len(r) == len(hdr)]
    ops = [(r[ix["Source"]].strip().split()[0] if not r[ix["Source"]].strip().startswith("@")
            else r[ix["Source"]].strip().split()[1]) for r in R]
    hot_idx = [i for i, o in enumerate(ops) if o.split(".")[0] == hot]
    lo, hi = (hot_idx[0], hot_idx[-1]) if hot_idx else (0, len(R) - 1)
    tot = defaultdict(float)
    region = {"hot": defaultdict(float), "other": defaultdict(float)}
    for i, r in enumerate(R):
        key = "hot" if lo <= i <= hi else "other"
        for s in stalls:
            v = float(r[ix[s]] or 0)
            tot[s] += v
            region[key][s] += v
    T = sum(tot.values()) or 1
    for key in ("hot", "other"):
        d = region[key]
        S = sum(d.values())
        print(f"{key:5s} region: {S / T:6.1%} of all samples; " +
              ", ".join(f"{k[6:]} {v / T:.1%}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:7]))


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
