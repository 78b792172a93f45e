"""Summarise an `ncu --page raw --csv` export: per kernel time, DRAM bytes, occupancy, issue
rate, top warp-stall reasons.  python tools/ncu_summary.py gpurun_out/x_raw.csv"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW"),
        ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
        ("smsp__inst_executed.sum", "inst")]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        print(r[idx["Kernel Name"]][:90])
        print("   " + "  ".join(f"{short}={r[idx[k]]}{units[idx[k]]}" for k, short in KEYS if k in idx))
        top = sorted(((float(r[idx[h]] or 0), h) for h in stall), reverse=True)[:5]
        print("   stalls: " + ", ".join(f"{h[34:-23]}={v:.2f}" for v, h in top))


if __name__ == "__main__":
    main(sys.argv[1])
