"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
python scripts/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches_summary.txt

Lists our kernels (namespace tg::) with launch count, mean duration and share of
our kernels' total time.  ncu times are cold-cache and serialised: compare
shares, not absolutes."""
import collections
import csv
import sys


def main(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum" or "tg::" not in r["Kernel Name"]:
            continue
        name = r["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(r["Metric Unit"], 1.0)
        us = float(r["Metric Value"].replace(",", "")) * scale
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values()) or 1.0
    print("# launch list summary (ncu --metrics gpu__time_duration.sum --clock-control none;")
    print("# cold-cache, serialised); our kernels only; share = of our kernels' time")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:<48} n={n:4d} mean={t / n:11.3f} us share={100 * t / total:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1])
