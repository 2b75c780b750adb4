"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launch count and mean / total device time (ms).
Times are cold-cache and serialised (ncu), so compare SHARES, not absolutes."""
import collections
import csv
import re
import sys


def main(path):
    agg = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.search(r"(\w+kernel\w*)", name)
        key = m.group(1) if m else name[:50]
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
            r["Metric Unit"], 1e-6)
        agg.setdefault(key, []).append(v)
    total = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8} {'mean ms':>10} {'total ms':>10} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):10.3f} {sum(v):10.3f} {sum(v) / total:6.1%}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
