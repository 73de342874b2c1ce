"""Top warp-stall SASS lines of one ncu report (run here, no GPU):
  python tools/ncu_top_sass.py <report.ncu-rep> [min_pct]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    lo = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    body = rows[2:]

    def f(r, k):
        try:
            return float(r[idx[k]].replace(",", ""))
        except (ValueError, KeyError, IndexError):
            return 0.0

    key = "Warp Stall Sampling (All Samples)"
    tot = sum(f(r, key) for r in body) or 1.0
    for i, r in enumerate(body):
        s = f(r, key) / tot * 100
        if s >= lo:
            print(f"{s:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']][:64]:64s} | prev {body[i - 1][idx['Source']][:48]}")


if __name__ == "__main__":
    main()
