"""Attribute long-scoreboard stall samples to the memory instruction that produced the waited-on
register (backward scan in the SASS listing).  python tools/ncu_longsb.py sass.csv [N]"""
import csv
import re
import sys
from collections import defaultdict


def main(path, n=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    if len(body) % 2 == 0 and body[: len(body) // 2] == body[len(body) // 2:]:
        body = body[: len(body) // 2]
    col = hdr.index("stall_long_sb")
    tot = sum(float(r[col] or 0) for r in body) or 1
    by_src = defaultdict(float)
    for k, r in enumerate(body):
        v = float(r[col] or 0)
        if v <= 0:
            continue
        text = r[1]
        srcs = re.findall(r"\bR(\d+)\b", text.split(",", 1)[1] if "," in text else "")
        found = None
        for j in range(k - 1, max(-1, k - 400), -1):
            t = body[j][1]
            op = t.split()[0] if not t.split()[0].startswith("@") else t.split()[1]
            if any(x in op for x in ("LDG", "LD.", "LDL", "LDS", "ATOM", "LDSM")) or op in ("LD",):
                dst = re.findall(r"\bR(\d+)\b", t)
                if dst and dst[0] in srcs:
                    found = f"{op} @{j}"
                    break
        by_src[found or "?"] += v
    print(f"long_sb samples {tot:.0f}")
    for key, v in sorted(by_src.items(), key=lambda kv: -kv[1])[:n]:
        j = int(key.split("@")[1]) if "@" in key else None
        ctx = body[j][1].strip()[:70] if j is not None else ""
        print(f"{100 * v / tot:5.1f}%  {key:28s} {ctx}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
