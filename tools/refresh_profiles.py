"""Refresh the profiles/ files that tools/r02_final.sh feeds (run here after
the GPU call merged gpurun_out/): bench lines, the roofline traffic record,
the bench launch list.

    python tools/refresh_profiles.py
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    for src, dst in (("fin_bench.json", "r02_bench_line.json"),
                     ("fin_bench_ref.json", "r02_bench_reference_line.json")):
        line = open(os.path.join(G, src)).read().strip().splitlines()[-1]
        json.loads(line)
        open(os.path.join(P, dst), "w").write(line + "\n")
    t = open(os.path.join(G, "fin_k_stiff3_raw.csv")).read()
    rows = list(csv.reader(io.StringIO(t[t.index('"ID"'):])))
    h, u, r = rows[0], rows[1], rows[2]
    ix = {k: i for i, k in enumerate(h)}

    def val(k):
        return float(r[ix[k]].replace(",", "")) * SCALE.get(u[ix[k]], 1.0)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    rec = {"kernel": "void k_stiff3<0, 128, false> (solver variant SF_IN_MASKED)",
           "workload": "16384x8192 cells (134M cells, 268,484,610 DOFs), tools/prof_matvec.py 16384 8192 3 1",
           "capture": "ncu --set full --clock-control none --import-source on -k regex:k_stiff -s 2 -c 1 "
                      "(tools/r02_final.sh), exported with --page raw --csv on the box",
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "alg_bytes_per_launch": 5369495584,
           "ncu_duration": float(r[ix["gpu__time_duration.sum"]].replace(",", "")),
           "ncu_duration_unit": u[ix["gpu__time_duration.sum"]],
           "registers_per_thread": int(r[ix["launch__registers_per_thread"]]),
           "dram_over_alg": (rd + wr) / 5369495584}
    json.dump(rec, open(os.path.join(P, "r02_roofline_traffic.json"), "w"), indent=1)
    head = ("# bench.py --steps 20 --warmup 3 --no-cpu --no-sweep --no-sharded under ncu -c 4000 "
            "--metrics gpu__time_duration.sum --clock-control none (tools/r02_final.sh): the launch "
            "list of the first 4000 launches (set-up, roofline matvecs, C2 iterations).  Per-launch "
            "times are cold-cache and serialised.\n")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_launches.py"),
                          os.path.join(G, "fin_launches.csv")], capture_output=True, text=True)
    open(os.path.join(P, "r02_bench_launches.txt"), "w").write(head + out.stdout)
    with open(os.path.join(G, "fin_launches.csv")) as fi, open(os.path.join(P, "r02_bench_launches.csv"), "w") as fo:
        fo.write(fi.read())
    print("refreshed: bench lines, roofline traffic", round(rec["dram_over_alg"], 3), "launch list")


if __name__ == "__main__":
    main()
