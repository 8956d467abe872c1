"""Summarise an ncu launch list (ncu --metrics gpu__time_duration.sum --csv)
into per-kernel launches / total / mean / share of the listed time."""
import csv
import sys
from collections import defaultdict


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "ns"
        ms = v / 1e6 if unit in ("ns", "nsecond") else v / 1e3 if unit in ("us", "usecond") else v
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(x[1] for x in agg.values())
    print(f"# {title}")
    print("# cold-cache, serialised per-launch times: compare SHARES with bench.py's live event timing")
    print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'mean_ms':>9s} {'share':>6s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda z: -z[1][1]):
        print(f"{k[:60]:60s} {n:8d} {ms:10.2f} {ms / n:9.3f} {100 * ms / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu launch list")
