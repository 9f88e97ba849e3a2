import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time share per kernel."""
import csv
import re
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
    tot[name] += float(r["Metric Value"].replace(",", ""))
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {100 * v / all_ns:6.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_ns / 1e3:10.1f}")
