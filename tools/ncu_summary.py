"""Summarise an ncu report: per kernel time, DRAM bytes, occupancy, issue,
pipe utilisation and the top warp-stall reasons."""
import csv
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fmacyc%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankconf"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall_cols = [(i, h) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in data:
        name = r[hdr.index("Kernel Name")]
        m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
        short = (m.group(0) if m else name)[:110]
        vals = []
        for key, lab in METRICS:
            if key in hdr:
                vals.append(f"{lab}={r[hdr.index(key)]}")
        stalls = []
        for i, h in stall_cols:
            try:
                stalls.append((float(r[i]), h))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        top = ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.1f}"
                        for v, h in stalls[:5])
        print(short)
        print("   ", " ".join(vals))
        print("    stalls:", top)


if __name__ == "__main__":
    main(sys.argv[1])
