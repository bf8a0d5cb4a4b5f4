"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    n = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", d["Kernel Name"])
    n = re.sub(r"^void ", "", n).split("(")[0]
    v = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1)
    tot[n] += v
    cnt[n] += 1
T = sum(tot.values())
steps = max(1, cnt.get("k_sample", 1))
print(f"{'kernel':40s} {'launches':>8s} {'us/step':>9s} {'share':>6s} {'avg us':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:40]:40s} {cnt[k]:8d} {v / 1e3 / steps:9.1f} {v / T * 100:5.1f}% {v / cnt[k] / 1e3:8.1f}")
print(f"total per step {T / 1e3 / steps:.1f} us over {steps} steps")
