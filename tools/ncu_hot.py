"""Top stall-sampled SASS lines of an ncu report's source page:
python tools/ncu_hot.py report.ncu-rep [top_n] (needs ncu on PATH)."""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    si, ci = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = []
    for idx, r in enumerate(rows[hi + 1:]):
        try:
            data.append((float(r[si]), idx, r[ci].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1.0
    for v, idx, src in sorted(data, reverse=True)[:top]:
        print(f"{v / tot:6.3f} #{idx:5d} {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
