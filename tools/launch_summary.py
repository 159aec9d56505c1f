"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total device time and share.  Cold-cache and serialised
under ncu, so compare shares, not absolutes.
  python tools/launch_summary.py gpurun_out/ev1/launches.csv > profiles/r01_launches_summary.txt"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("(anonymous namespace)", "anon").replace("<unnamed>", "anon"))
    name = name.replace("esg::anon::", "").replace("esg::", "").replace("void ", "")
    return name.strip()


def main():
    path = sys.argv[1]
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = short(r[ki])
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + ms)
    total = sum(t for _, t in agg.values())
    print(f"# {path}: {sum(c for c, _ in agg.values())} launches, {total:.1f} ms device time (ncu, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg ms':>9s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {t:10.2f} {100 * t / total:6.1f}% {t / c:9.4f}")


if __name__ == "__main__":
    main()
