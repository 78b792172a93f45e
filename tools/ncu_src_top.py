"""Top CUDA source lines by a per-instruction metric (default warp-stall samples) from
`ncu --page source --csv --print-source cuda,sass` (SASS rows are charged to the CUDA line
above them).  python tools/ncu_src_top.py file.csv [N] [column]"""
import csv
import sys
from collections import defaultdict


def main(path, n=25, col="Warp Stall Sampling (All Samples)"):
    rows = list(csv.reader(open(path)))
    cur_file, hdr, line_key = None, None, None
    agg = defaultdict(float)
    text = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0]:
            line_key = f"{cur_file}:{r[0]}"
            text[line_key] = r[1].strip()[:100]
        try:
            v = float(r[hdr.index(col, 2)] or 0)  # the SASS-side column
        except (ValueError, IndexError):
            continue
        if line_key:
            agg[line_key] += v
    tot = sum(agg.values()) or 1
    print(f"total {col}: {tot:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
        print(f"{100 * v / tot:5.1f}%  {k:24s} {text.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)")
