"""Summarise an ncu report's source page: stall reasons overall and top instructions.
usage: python tools/ncu_stalls.py report.ncu-rep [kernel-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the page repeats per kernel instance; take the first block
hdr = rows[1]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
per = []
seen = set()
for r in rows[2:]:
    if len(r) != len(hdr):
        break
    addr = r[0]
    if addr in seen:
        break
    seen.add(addr)
    d = dict(zip(hdr, r))
    s = {k: int(d[k]) if d[k].isdigit() else 0 for k in reasons}
    for k, v in s.items():
        tot[k] += v
    per.append((sum(s.values()), d["Source"].strip(), s))
T = sum(tot.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]}={v*100/T:.1f}%" for k, v in tot.most_common(10)))
for n, src, s in sorted(per, key=lambda x: -x[0])[:20]:
    top = max(s, key=s.get)
    print(f"{n*100/T:5.1f}% {top[6:]:14s} {src[:90]}")
