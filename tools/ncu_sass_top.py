"""Top SASS instructions by stall samples from `ncu --page source --csv --print-source sass`,
with the dominant stall reasons and the preceding-instruction context.
python tools/ncu_sass_top.py file.csv [N]"""
import csv
import sys


def main(path, n=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    stall_cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[si] or 0) for r in body) or 1
    inst = sum(float(r[ie] or 0) for r in body)
    print(f"samples {tot:.0f}, warp instructions {inst / 1e6:.1f} M, {len(body)} SASS lines")
    # opcode totals of stall samples
    from collections import defaultdict
    byop = defaultdict(float)
    for r in body:
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        byop[op.split(".")[0]] += float(r[si] or 0)
    print("stall samples by opcode:", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in sorted(byop.items(), key=lambda kv: -kv[1])[:14]))
    order = sorted(range(len(body)), key=lambda k: -float(body[k][si] or 0))[:n]
    for k in order:
        r = body[k]
        st = sorted(((float(r[i] or 0), h) for i, h in stall_cols), reverse=True)[:2]
        print(f"{100 * float(r[si] or 0) / tot:4.1f}% [{k:5d}] {r[1].strip()[:60]:60s} {' '.join(f'{h}={v:.0f}' for v, h in st)}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
