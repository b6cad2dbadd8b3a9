"""Summarise an ncu --csv launch list: total time per kernel name."""
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    tot[name] += float(r["Metric Value"]) / 1e3; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.1f} {v/cnt[k]:9.2f} {100*v/T:5.1f}%")
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
