"""DRAM traffic per launch of the r2 kernels from an ncu metrics capture
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv; tools/gpu_profile_r2.sh):
  python tools/traffic_summary.py gpurun_out/<tag>/traffic.csv <run-tag> [config]
prints the per-kernel table (profiles/<round>_traffic_summary.txt) and rewrites profiles/traffic.json
(bytes per launch = read + write, averaged over the capture's launches), which bench.py's
roofline.traffic reads."""
import collections
import csv
import json
import os
import re
import sys


def main(path, tag, config="c3"):
    rows = list(csv.reader(open(path, errors="replace")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ni, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"(k2?_[a-z0-9_]+)", r[ki])
        if not m:
            continue
        d = per.setdefault(m.group(1), collections.defaultdict(float))
        d[r[ni]] += float(r[vi].replace(",", ""))
        d.setdefault("_ids", set())
        d["_ids"].add(r[idi]) if isinstance(d["_ids"], set) else None
    out = {}
    for k, d in per.items():
        n = len(d["_ids"])
        rd, wr = d["dram__bytes_read.sum"] / n, d["dram__bytes_write.sum"] / n
        ms = d["gpu__time_duration.sum"] / n / 1e6
        out[k] = rd + wr
        print(f"{k:12s} launches {n}  read {rd / 1e6:9.2f} MB  write {wr / 1e6:9.2f} MB  "
              f"{ms:9.3f} ms/launch  {(rd + wr) / 1e9 / (ms * 1e-3):9.1f} GB/s")
    jp = os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic.json")
    try:
        cur = json.load(open(jp))
    except Exception:
        cur = {}
    cur[config] = out
    cur["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum, one "
                      f"capture of tools/profile_step.py --config {config} --steps 1 (full size), "
                      f"tools/gpu_profile_r2.sh (run {tag}); bytes per launch averaged over the launches of "
                      "the capture; written by tools/traffic_summary.py")
    json.dump(cur, open(jp, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
