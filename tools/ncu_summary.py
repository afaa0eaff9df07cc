"""Summarise an ncu --set full report: per-kernel duration, DRAM bytes, throughput.

    python tools/ncu_summary.py report.ncu-rep|raw.csv [algorithmic_bytes_per_launch ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%pk"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%pk"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("lts__t_sector_hit_rate.pct", "l2_hit%"),
]


def main(path):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` exported on the GPU box
        out = open(path).read()
        out = out[out.index('"ID"'):] if '"ID"' in out else out
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0]
        vals = []
        for k, _ in KEYS:
            v = d.get(k, "")
            u = units[hdr.index(k)] if k in hdr else ""
            vals.append(f"{v} {u}".strip())
        print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
