"""Summarise ncu reports into profiles/: a markdown table of the hot kernels and
ncu_traffic.json (DRAM bytes per launch, used as bench.py's roofline.traffic)."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__t_sectors_op_read.sum", "L2 rd sectors"),
    ("lts__t_sectors_op_write.sum", "L2 wr sectors"),
    ("lts__t_sectors_op_atom.sum", "L2 atom sectors"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb / issue"),
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main(tag, reps):
    lines = [f"# ncu summary ({tag})", "", "Captured with `ncu --set full --clock-control none --import-source on` "
             "(cold cache, serialised replays: compare shares, not absolutes).", ""]
    lines.append("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    lines.append("|---" * (len(METRICS) + 1) + "|")
    traffic = {}
    for rep in reps:
        for row, units in raw(rep):
            name = row["Kernel Name"].split("(")[0].replace("void ", "").replace("hive::", "")
            short = name.split("<")[0]
            vals = []
            for m, _ in METRICS:
                v = row.get(m, "")
                u = units.get(m, "")
                vals.append(f"{v} {u}".strip())
            lines.append(f"| {name} | " + " | ".join(vals) + " |")
            try:
                rd = float(row["dram__bytes_read.sum"]) * (1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1e6 if units["dram__bytes_read.sum"] == "Mbyte" else 1)
                wr = float(row["dram__bytes_write.sum"]) * (1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1e6 if units["dram__bytes_write.sum"] == "Mbyte" else 1)
                traffic.setdefault(short, rd + wr)
            except (KeyError, ValueError):
                pass
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))
    print(json.dumps(traffic))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
