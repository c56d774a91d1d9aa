"""Summarise ncu reports into profiles/: a markdown table of the hot kernels and
ncu_traffic.json (DRAM bytes per launch, used as bench.py's roofline.traffic).

Usage: python tools/ncu_summary.py TAG [--ops kernel=N ...] report.ncu-rep ...
--ops gives the operations one launch of a kernel processed, for the per-op
columns (DRAM bytes / op, L2 sectors / op, atomics / s).  The L2 sector
counters are not part of `--set full` on this ncu / Blackwell: the capture must
add them with `--metrics` (tools/ncu_run.sh does)."""
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
    ("lts__t_sectors_op_red.sum", "L2 red sectors"),
    ("lts__t_requests_op_atom.sum", "L2 atom requests"),
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


L2_METRICS = ("lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,"
              "lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "Ksector": 1e3, "Msector": 1e6,
         "Gsector": 1e9, "request": 1, "Krequest": 1e3, "Mrequest": 1e6, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "": 1}


def num(row, units, m):
    v = row.get(m, "")
    if v in ("", "n/a"):
        return None
    return float(v.replace(",", "")) * SCALE.get(units.get(m, ""), 1)


def main(tag, reps, ops=None, write_traffic=True):
    ops = ops or {}
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
    per_op = ["", "Per operation (ops per launch given to the tool):", "",
              "| kernel | ops | DRAM B/op | L2 rd sectors/op | L2 wr sectors/op | L2 atom sectors/op | "
              "L2 red sectors/op | atomics G/s |", "|---|---|---|---|---|---|---|---|"]
    for rep in reps:
        for row, units in raw(rep):
            name = row["Kernel Name"].split("(")[0].replace("void ", "").replace("hive::", "")
            short = name.split("<")[0]
            n = ops.get(short)
            if not n:
                continue
            t = num(row, units, "gpu__time_duration.sum")
            d = (num(row, units, "dram__bytes_read.sum") or 0) + (num(row, units, "dram__bytes_write.sum") or 0)
            f = lambda m: (lambda x: "" if x is None else f"{x / n:.3f}")(num(row, units, m))
            at = num(row, units, "lts__t_requests_op_atom.sum")
            per_op.append(f"| {name} | {n} | {d / n:.1f} | {f('lts__t_sectors_op_read.sum')} | "
                          f"{f('lts__t_sectors_op_write.sum')} | {f('lts__t_sectors_op_atom.sum')} | "
                          f"{f('lts__t_sectors_op_red.sum')} | "
                          f"{'' if at is None or not t else f'{at / t / 1e9:.1f}'} |")
    lines += per_op
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    if write_traffic:   # the cfg2 step kernels' DRAM bytes: bench.py's roofline.traffic source
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))
    print(json.dumps(traffic))


if __name__ == "__main__":
    args = sys.argv[2:]
    ops, reps = {}, []
    i = 0
    while i < len(args):
        if args[i] == "--ops":
            k, v = args[i + 1].split("=")
            ops[k] = int(v)
            i += 2
        elif args[i] == "--no-traffic":
            i += 1
        else:
            reps.append(args[i])
            i += 1
    main(sys.argv[1], reps, ops, write_traffic="--no-traffic" not in sys.argv)
