"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
  python tools/launch_summary.py gpurun_out/<tag>/launches.csv > profiles/<round>_launches_summary.csv
share = fraction of all GPU time of the command (setup, warm-up, diagnostics, timed and e2e steps)."""
import collections
import csv
import sys


def main(p):
    rows = list(csv.reader(open(p)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        try:
            v = float(r[mi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0]
        tot[k] += v
        cnt[k] += 1
    T = sum(tot.values())
    print("# ncu launch list, gpu__time_duration.sum; per-launch times are cold-cache and serialised")
    print("kernel,launches,total_ms,share_pct,per_launch_us")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f'"{k}",{cnt[k]},{v / 1e6:.3f},{100 * v / T:.2f},{v / cnt[k] / 1e3:.1f}')


if __name__ == "__main__":
    main(sys.argv[1])
