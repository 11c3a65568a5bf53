"""Summarise an ncu --metrics gpu__time_duration.sum launch list.

    python scripts/launches.py gpurun_out/launches.csv [--half]   (--half: second half only)
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
mi = hdr.index("Metric Name")
data = [r for r in data if r[mi] == "gpu__time_duration.sum"]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
seq = [(r[ki].split("(")[0].replace("void ", "").replace("pmf::", ""),
        float(r[vi].replace(",", "")) * scale[r[ui]]) for r in data]
if "--half" in sys.argv:
    seq = seq[len(seq) // 2:]
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, us in seq:
    tot[k] += us
    cnt[k] += 1
T = sum(tot.values())
print(f"{len(seq)} launches, {T / 1e3:.3f} ms of kernel time")
print("| kernel | launches | total ms | share | avg us |")
print("|---|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| {k} | {cnt[k]} | {tot[k] / 1e3:.3f} | {100 * tot[k] / T:.1f}% | {tot[k] / cnt[k]:.1f} |")
