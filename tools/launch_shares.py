"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
        name = re.sub(r"cpb::", "", name)
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':42s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:42]:42s} {cnt[k]:8d} {v:12.1f} {v / s:7.3f}")
    print(f"{'TOTAL':42s} {sum(cnt.values()):8d} {s:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
