"""Summarise an ncu --set full report: per kernel SOL, occupancy, stalls, dram bytes.
Usage: python tools/ncu_summary.py report.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEEP = {
    "GPU Speed Of Light Throughput": ["Duration", "Compute (SM) Throughput", "Memory Throughput",
                                      "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput"],
    "Occupancy": ["Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM"],
    "Launch Statistics": ["Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block"],
    "Scheduler Statistics": ["Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler"],
    "Memory Workload Analysis": ["L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction"],
}


def main(rep, out=None):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    res = {}
    for d in csv.DictReader(io.StringIO(det)):
        key = f'{d["ID"]}:{d["Kernel Name"].split("(")[0]}'
        e = res.setdefault(key, {})
        if d["Metric Name"] in KEEP.get(d["Section Name"], []):
            e[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    rows = list(csv.reader(io.StringIO(raw)))
    if rows:
        h = rows[0]
        want = [c for c in h if c in ("dram__bytes_read.sum", "dram__bytes_write.sum")
                or c.startswith("smsp__pcsamp_warps_issue_stalled_")]
        for r in rows[2:]:
            d = dict(zip(h, r))
            key = f'{d["ID"]}:{d["Kernel Name"].split("(")[0]}'
            e = res.setdefault(key, {})
            for c in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if c in d:
                    e[c] = d[c] + " " + rows[1][h.index(c)]
            stalls = {}
            for c in want:
                if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued"):
                    try:
                        stalls[c.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[c].replace(",", ""))
                    except ValueError:
                        pass
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
            e["top_stalls_frac"] = {k: round(v / tot, 3) for k, v in top}
    txt = json.dumps(res, indent=1)
    if out:
        open(out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main(*sys.argv[1:])
