"""Instruction mix and stall samples per opcode from an ncu source page
(`--page source --csv --print-source sass`, tools/src_ncu.sh).

    python tools/sass_mix.py SRC_sass.csv CELLS [--groups]
"""
import collections
import csv
import re
import sys


def main(path, cells, groups=False):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    tot = 0
    byop, samp, wait = collections.Counter(), collections.Counter(), collections.Counter()
    counts = collections.Counter()
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        src = r[ix["Source"]].strip()
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0].split(".")[0]
        byop[op] += n
        samp[op] += s
        wait[op] += int(r[ix["stall_wait"]] or 0)
        counts[n] += 1
        tot += n
    print(f"warp instructions {tot}, per cell {tot * 32 / cells:.1f}, samples {sum(samp.values())}")
    for k, v in byop.most_common(25):
        print(f"  {k:12s} {v / tot * 100:5.1f}%  inst/cell {v * 32 / cells:6.1f}  samples {samp[k]:6d}  wait {wait[k]}")
    if groups:
        print("execution-count groups (count: instructions):")
        for n, c in sorted(counts.items(), key=lambda kv: -kv[0] * kv[1])[:8]:
            print(f"  {n}: {c}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), "--groups" in sys.argv)
