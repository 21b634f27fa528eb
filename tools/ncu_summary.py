"""Summarise an ncu --set full report: per-launch duration, DRAM traffic,
tensor / issue activity, occupancy.  usage: python tools/ncu_summary.py REP [title]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "int8 MMA subpipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"### {title}\n")
    print("| launch | kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|---" * (2 + len(METRICS)) + "|")
    for k, r in enumerate(data):
        name = r[col.get("Kernel Name", 4)].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        vals = []
        for m, _ in METRICS:
            i = col.get(m)
            vals.append(f"{r[i]} {units[i]}".strip() if i is not None else "n/a")
        print(f"| {k} | {name} | " + " | ".join(vals) + " |")
    print()


if __name__ == "__main__":
    main()
