"""Per-kernel stall-reason totals and executed-instruction mix by opcode from
`ncu --page source --csv --print-source cuda,sass`.  python tools/ncu_sass_stats.py file.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    stall = defaultdict(float)
    ops = defaultdict(float)
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[2]:
            continue
        sass = r[3].strip()
        try:
            n = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        op = sass.split()[0] if sass else "?"
        if op.startswith("@"):
            op = sass.split()[1]
        ops[op.split(".")[0]] += n
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stall[h] += float(r[i] or 0)
                except ValueError:
                    pass
    ts = sum(stall.values()) or 1
    print("stalls:", ", ".join(f"{k[6:]}={100 * v / ts:.1f}%" for k, v in sorted(stall.items(), key=lambda kv: -kv[1])[:9]))
    to = sum(ops.values()) or 1
    print(f"warp instructions: {to / 1e6:.1f} M;", ", ".join(f"{k}={100 * v / to:.1f}%" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:22]))


if __name__ == "__main__":
    main(sys.argv[1])
