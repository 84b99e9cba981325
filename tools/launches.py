"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
total = 0.0
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        ns = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        us = ns / 1000.0 if unit == "ns" else ns * (1000.0 if unit == "ms" else 1.0) if unit != "us" else ns
        name = d["Kernel Name"].split("(")[0]
        per.setdefault(name, []).append(us)
        total += us
for name, v in per.items():
    print("%-45s n=%-3d mean %9.1f us  share %5.1f%%" % (name[:45], len(v), sum(v) / len(v), 100 * sum(v) / total))
print("total %.1f us over %d launches" % (total, sum(len(v) for v in per.values())))
