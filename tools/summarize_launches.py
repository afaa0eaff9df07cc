"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/summarize_launches.py launches.csv [label]
Prints per-kernel count, mean duration (us) and share of the summed time.
"""
import collections
import csv
import sys


def main(path, label=""):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d.get("Metric Unit"), 1e-3)
                name = d["Kernel Name"].split("(")[0]
                data[name].append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in data.values())
    print(f"# {label} launch list: {sum(len(v) for v in data.values())} launches, {tot:.1f} us total")
    print(f"{'kernel':52s} {'n':>5s} {'mean_us':>9s} {'share':>7s}")
    for k, v in sorted(data.items(), key=lambda x: -sum(x[1])):
        print(f"{k:52s} {len(v):5d} {sum(v) / len(v):9.2f} {sum(v) / tot * 100:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
