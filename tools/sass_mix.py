"""Dynamic instruction mix from an ncu source page (SASS): executed warp-instructions per opcode,
split by pipe class, plus the share of each opcode.  python tools/sass_mix.py <src.csv>"""
import csv
import sys
from collections import Counter

FMA = {"FFMA", "FMUL", "FADD", "FFMA2", "FMUL2", "FADD2", "IMAD", "HFMA2", "FSWZADD", "IDP", "IMUL"}


def main(p):
    rows = list(csv.reader(open(p)))
    hdr = rows[1]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    cnt, tot = Counter(), 0
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        src = r[isrc].strip()
        if src.startswith("@"):
            src = src.split(None, 1)[1]
        op = src.split()[0] if src else "?"
        base = op.split(".")[0]
        full = op if base == "IMAD" else base
        n = int(r[iex] or 0)
        cnt[full] += n
        tot += n
    fma = sum(v for k, v in cnt.items() if k.split(".")[0] in FMA)
    dbl = sum(v for k, v in cnt.items() if k in ("FFMA2", "FADD2", "FMUL2"))
    print(f"total warp-inst {tot:.4g}; FMA-pipe {fma:.4g} ({fma / tot:.1%}); packed f32x2 {dbl:.4g}")
    print(f"FMA-pipe cycles (f32x2 = 2): {fma + dbl:.4g}; useful share of FMA instr: "
          f"{cnt['FFMA2'] + cnt['FADD2']:.4g}")
    for k, v in cnt.most_common(30):
        print(f"  {k:24s} {v:14.4g}  {v / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
