"""Turn the round-2 final captures (gpurun_out/r02z_*) into the committed
profiles/: per-kernel ncu summaries, launch lists, DRAM traffic per launch
(profiles/ncu_traffic.json, copied by bench.py into roofline.traffic)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
SRC = os.path.join(ROOT, "gpurun_out")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02z"

sys.path.insert(0, os.path.join(ROOT, "tools"))
import launches  # noqa: E402

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def summary(name, title, notes):
    rep = os.path.join(SRC, f"{TAG}_{name}.ncu-rep")
    if not os.path.exists(rep):
        print("missing", rep)
        return None
    h, u, data = raw(rep)
    r = data[0]
    lines = [f"# {title}", "", "Command (one B200; the plain command exited 0 before the ncu run of the same command line, "
             "tools/prof.sh): `ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ "
             f"-k regex:... -c 1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline ...` ({TAG}_{name}.ncu-rep)", "",
             "| metric | value |", "|---|---|"]
    lines.append(f"| kernel | `{r[h.index('Kernel Name')].split('(')[0]}` |")
    stalls = []
    for i, n in enumerate(h):
        if "pcsamp_warps_issue_stalled" in n and "not_issued" not in n:
            stalls.append((int(float(r[i] or 0)), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    for m, label in WANT:
        if m in h:
            i = h.index(m)
            lines.append(f"| {label} | {r[i]} {u[i]} |")
    tot = sum(s for s, _ in stalls) or 1
    top = ", ".join(f"{n} {100.0 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:7])
    lines.append(f"| warp-state samples (top) | {top} |")
    lines += ["", notes, ""]
    rd = to_bytes(r[h.index("dram__bytes_read.sum")], u[h.index("dram__bytes_read.sum")])
    wr = to_bytes(r[h.index("dram__bytes_write.sum")], u[h.index("dram__bytes_write.sum")])
    return "\n".join(lines), int(rd + wr)


def main():
    traffic = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the dominant kernel from one `ncu --set "
                        "full --clock-control none` capture per config (tools/prof.sh, tools/final_r02.sh); bench.py copies it "
                        "into roofline.traffic"}
    try:
        traffic.update({k: v for k, v in json.load(open(os.path.join(OUT, "ncu_traffic.json"))).items() if k != "_note"})
    except Exception:
        pass
    specs = [
        ("scan4tc_cfg4", "r02 final -- Quick ADC tcgen05 filter, cfg4 shard (125M codes x 10,000 queries): the default bench kernel",
         "scan4tc_kernel_cfg4", NOTES.get("scan4tc_cfg4", "")),
        ("scan8p_cfg0", "r02 final -- packed float filter (scan8p, resident tables), cfg0 (1M x 8x8, 1,000 queries)",
         "scan8p_kernel_cfg0", NOTES.get("scan8p_cfg0", "")),
        ("scan8p_cfg2", "r02 final -- packed float filter (scan8p, streamed quads), cfg2 (1M x 64x8, 1,000 queries)",
         "scan8p_kernel_cfg2", NOTES.get("scan8p_cfg2", "")),
        ("list8_cfg3", "r02 final -- packed IVF list scan (ivf_list8_kernel), cfg3 (1e8 codes, K = 65,536, nprobe 64, 10,000 queries)",
         "ivf_list8_kernel", NOTES.get("list8_cfg3", "")),
    ]
    for name, title, key, notes in specs:
        res = summary(name, title, notes)
        if res is None:
            continue
        text, nbytes = res
        lst = os.path.join(SRC, f"{TAG}_launches_{name.split('_')[-1]}.csv")
        if os.path.exists(lst):
            text += "\n## Launch list of one search (ncu gpu__time_duration, cold-cache and serialised: shares, not absolutes)\n\n```\n" + \
                    launches.summarise(lst) + "\n```\n"
            shutil.copy(lst, os.path.join(OUT, f"r02_final_launches_{name.split('_')[-1]}.csv"))
        open(os.path.join(OUT, f"r02_final_{name}.md"), "w").write(text)
        traffic[key] = {"bytes": nbytes, "round": 2, "capture": f"profiles/r02_final_{name}.md",
                        "note": TRAFFIC_NOTES.get(name, "")}
        print(name, nbytes)
    lst = os.path.join(SRC, f"{TAG}_launches_cfg1.csv")
    if os.path.exists(lst):
        shutil.copy(lst, os.path.join(OUT, "r02_final_launches_cfg1.csv"))
    json.dump(traffic, open(os.path.join(OUT, "ncu_traffic.json"), "w"), indent=1)


NOTES = {}
TRAFFIC_NOTES = {
    "scan4tc_cfg4": "one main-range launch = 1/60 of the search (16,208 tiles: 16.6 MB of codes + 40 groups x 72 KB of tables "
                    "= 19.5 MB algorithmic); the search's ~61 filter launches read ~1.2 GB for 1.0 GB of codes",
    "scan8p_cfg0": "the second filter launch (7/8 of the tiles: 7 MB of codes + 4 MB of packed tables algorithmic)",
    "scan8p_cfg2": "the second filter launch (7/8 of the tiles: 56 MB of codes + 32 MB of packed tables algorithmic, plus "
                   "the candidate writes)",
    "list8_cfg3": "the one list-scan launch of a search: 0.8 GB of codes + 0.5 GB of per-list W tables algorithmic, plus U "
                  "tables that miss L2 and the candidate writes",
}
if __name__ == "__main__":
    np = os.path.join(ROOT, "tools", "profile_notes_r02.json")
    if os.path.exists(np):
        NOTES = json.load(open(np))
    main()
