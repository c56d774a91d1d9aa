"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
markdown table: launches, total and mean time and share per kernel."""
import collections, csv, re, sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    agg = collections.defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("hive::", "")
        if not name.startswith("k_"):
            name = "torch / memset (bench plumbing)"
        agg[name].append(float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]])
    return agg


def main(path, title):
    agg = load(path)
    tot = sum(sum(v) for v in agg.values())
    out = [f"# {title}", "", "Cold-cache, serialised launches (ncu `gpu__time_duration.sum`, `--clock-control none`): "
           "compare each kernel's SHARE with the event-timed numbers, not the absolutes.", "",
           "| kernel | launches | total ms | mean us | max us | share |", "|---|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| {k} | {len(v)} | {sum(v):.3f} | {1e3 * sum(v) / len(v):.1f} | {1e3 * max(v):.1f} | "
                   f"{100 * sum(v) / tot:.1f}% |")
    out.append(f"| **total** | {sum(len(v) for v in agg.values())} | {tot:.3f} | | | 100% |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
