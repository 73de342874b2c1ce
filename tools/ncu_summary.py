"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>   per-kernel share of device time
  python tools/ncu_summary.py full <report.ncu-rep|raw.csv>  key metrics per captured launch
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(path, after=None, seq=False):
    """after: only launches following the last launch whose name starts with it"""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    body = rows[hi + 1:]
    if after:
        last = max(i for i, r in enumerate(body) if len(r) > ki and r[ki].replace("void ", "").startswith(after))
        body = body[last + 1:]
    if seq:
        for r in body:
            if len(r) > vi and r[vi]:
                print(f"{float(r[vi].replace(',', '')) * UNIT.get(r[ui], 1.0):10.1f} us  {r[ki][:90]}  grid={r[h.index('Grid Size')]}")
    for r in body:
        if len(r) <= vi or not r[vi]:
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")[:60]
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    print(f"| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v/1e3:.2f} | {100*v/T:.1f}% | {v/cnt[k]:.1f} |")
    print(f"\ntotal device time {T/1e3:.2f} ms over {sum(cnt.values())} launches")


METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall lsb"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch"),
]


def full(path):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` exported on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = {n: i for i, n in enumerate(h)}
    print("| kernel | " + " | ".join(m[1] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        cells = [r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:45]]
        for m, _ in METRICS:
            v = r[idx[m]] if m in idx else "-"
            u = units[idx[m]] if m in idx else ""
            cells.append(f"{v} {u}".strip())
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None, "--seq" in sys.argv)
    else:
        full(sys.argv[2])
