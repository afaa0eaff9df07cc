"""Markdown tables from ncu CSV exports (the files the r02 evidence runs bring
back in gpurun_out/).

    python tools/summarize_metrics.py raw    REPORT_raw.csv   [--E cells]
    python tools/summarize_metrics.py launch METRICS.csv      [--iteration K]

raw:    `ncu --page raw --csv` (one row per launch): duration, DRAM bytes and
        GB/s, instructions per cell, issue activity, warps, registers.
launch: `ncu --csv --metrics ...` (one row per metric): per-kernel totals over
        iteration K of the run (iterations split at k_filter_fwd4 launches),
        plus the first (fine-level) launch of every kernel.
"""
import collections
import csv
import io
import sys

PEAK = 6548.2  # MEASURED_PEAKS.json hbm_gbs of this pool


def _csv(path):
    text = open(path).read()
    return text[text.index('"ID"'):]


def _short(name):
    return name.split("(")[0].replace("<unnamed>::", "").replace("bsp::", "").replace("void ", "")


_SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(path, cells):
    rows = list(csv.reader(io.StringIO(_csv(path))))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}

    def get(r, k, default=""):
        return r[ix[k]] if k in ix else default

    def val(r, k):  # ms for times, bytes for sizes
        v = float(get(r, k).replace(",", ""))
        return v * _SCALE.get(units[ix[k]], 1.0)

    print("| kernel | ms | DRAM GB | GB/s | of peak | inst/cell | issue % | warps % | regs |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        ms = val(r, "gpu__time_duration.sum")
        b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        inst = get(r, "smsp__inst_executed.sum")
        ipc = f"{float(inst.replace(',', '')) * 32 / cells:.1f}" if inst and cells else ""
        print(f"| {_short(get(r, 'Kernel Name'))} | {ms:.4f} | {b / 1e9:.3f} | "
              f"{b / (ms * 1e-3) / 1e9:.0f} | {b / (ms * 1e-3) / 1e9 / PEAK:.2f} | {ipc} | "
              f"{get(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
              f"{get(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')} | "
              f"{get(r, 'launch__registers_per_thread')} |")


def launch(path, iteration):
    rows = list(csv.DictReader(io.StringIO(_csv(path))))
    launches = collections.OrderedDict()
    for r in rows:
        d = launches.setdefault(int(r["ID"]), {"name": _short(r["Kernel Name"]),
                                               "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    L = list(launches.values())
    starts = [i for i, d in enumerate(L) if d["name"].startswith("k_filter_fwd4")]
    it = L[starts[iteration]:starts[iteration + 1]] if len(starts) > iteration + 1 else \
        L[starts[iteration]:]
    agg = collections.OrderedDict()
    for d in it:
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"] / 1e6
        a[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    print(f"iteration {iteration}: {len(it)} launches, "
          f"{sum(a[1] for a in agg.values()):.3f} ms serialised\n")
    print("| kernel | launches | ms | DRAM GB | GB/s | of peak |")
    print("|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        g = a[2] / (a[1] * 1e-3) / 1e9
        print(f"| {k} | {a[0]} | {a[1]:.3f} | {a[2] / 1e9:.3f} | {g:.0f} | {g / PEAK:.2f} |")
    print("\nfirst launch of each kernel (the fine level for the multigrid kernels):\n")
    print("| kernel | grid | ms | DRAM GB | GB/s | of peak |")
    print("|---|---|---|---|---|---|")
    seen = set()
    for d in it:
        if d["name"] in seen:
            continue
        seen.add(d["name"])
        ms = d["gpu__time_duration.sum"] / 1e6
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        g = b / (ms * 1e-3) / 1e9
        print(f"| {d['name']} | {d['grid']} | {ms:.4f} | {b / 1e9:.3f} | {g:.0f} | {g / PEAK:.2f} |")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "raw":
        E = int(sys.argv[sys.argv.index("--E") + 1]) if "--E" in sys.argv else 0
        raw(path, E)
    else:
        k = int(sys.argv[sys.argv.index("--iteration") + 1]) if "--iteration" in sys.argv else 1
        launch(path, k)
