"""Per-kernel table of the LAST hx_rotate in an ncu launch list of
`tools/prof.py ks B` (metrics: time, dram bytes, FP64 pipe %, issue %)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        e = L.setdefault(d["ID"], {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    hx = [v for v in L.values() if "hx::" in v["name"]]
    # the last rotate: everything after the combine (fused or not) that ends
    # the previous key switch, i.e. the last combine before the last inner product
    last_in = max(i for i, v in enumerate(hx) if "ks_inner" in v["name"])
    prev = [i for i, v in enumerate(hx[:last_in]) if "combine" in v["name"]]
    start = prev[-1] + 1 if prev else 0
    seq = hx[start:]
    tot = sum(v["gpu__time_duration.sum"] for v in seq)
    print(f"{'kernel':58s} {'ms':>7s} {'share':>6s} {'GB':>6s} {'TB/s':>5s} {'fp64%':>6s} {'issue%':>6s}")
    for v in seq:
        t = v["gpu__time_duration.sum"]
        gb = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e9
        print(f"{v['name'][:58]:58s} {t / 1e6:7.3f} {100 * t / tot:5.1f}% {gb:6.2f} {gb / (t / 1e9) / 1e3:5.2f} "
              f"{v.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):6.1f} "
              f"{v.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):6.1f}")
    print(f"total {tot / 1e6:.2f} ms over {len(seq)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
