"""ncu --set full report(s) -> a markdown table of the counters each kernel's design is
judged by (SM / FP64 / tensor pipes, L1 / L2 hit rates, L2 and DRAM throughput, occupancy,
top stall). Usage: python tools/ncu_table.py out.md report1.ncu-rep [report2 ...]"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "time us", 1, "us"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1, ""),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1, ""),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1, ""),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %", 1, ""),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %", 1, ""),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1, ""),
    ("lts__t_sectors.sum.per_second", "L2 GB/s", 32.0, ""),  # sectors/ns x 32 B = GB/s
    ("dram__bytes.sum.per_second", "DRAM GB/s", 1e-9, ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1, ""),
]
UNIT = {"Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6, "byte/s": 1, "usecond": 1e-6, "msecond": 1e-3,
        "nsecond": 1e-9, "%": 1, "": 1}


def num(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    if u in ("us", "usecond"):
        return x
    if u in ("ms", "msecond"):
        return x * 1e3
    if u in ("ns", "nsecond"):
        return x * 1e-3
    return x * UNIT.get(u, 1)


def rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        out = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")}
        for key, name, scale, _ in COLS:
            if key in d:
                v = num(d[key], units[h.index(key)])
                out[name] = None if v is None else v * scale
        stalls = {c.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(d[c], "") or 0.0 for c in h
                  if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        k, v = max(stalls.items(), key=lambda kv: kv[1]) if stalls else ("-", 0)
        out["top stall"] = f"{k} {100 * v / tot:.0f}%"
        yield out


def main(dst, *reps):
    hdr = ["kernel"] + [c[1] for c in COLS] + ["top stall"]
    lines = ["| " + " | ".join(hdr) + " |", "|" + "---|" * len(hdr)]
    for rep in reps:
        for o in rows(rep):
            cells = [o["kernel"][:48]]
            for _, name, _, _ in COLS:
                v = o.get(name)
                cells.append("-" if v is None else (f"{v:.1f}" if name != "time us" else f"{v:.0f}"))
            cells.append(o["top stall"])
            lines.append("| " + " | ".join(cells) + " |")
    txt = "\n".join(lines) + "\n"
    open(dst, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main(*sys.argv[1:])
