"""Summarise an ncu --csv launch list: total time (and DRAM bytes, when the
list carries dram__bytes_read/write.sum) per kernel name; with --sweep, also
the DRAM traffic of the dense sweep's launches (k_gemm / k_potrf_diag /
k_panel_take*) and their share of the step."""
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
per = collections.defaultdict(dict)
for r in rows:
    per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = collections.defaultdict(float); byt = collections.defaultdict(float); cnt = collections.Counter()
for (i, name), m in per.items():
    k = name.split("(")[0]
    tot[k] += m.get("gpu__time_duration.sum", 0.0) / 1e3
    byt[k] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    cnt[k] += 1
T = sum(tot.values())
has_b = any(byt.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}" + (f" {'DRAM MB':>9s} {'GB/s':>7s}" if has_b else ""))
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    line = f"{k[:60]:60s} {cnt[k]:8d} {v:10.1f} {v/cnt[k]:9.2f} {100*v/T:5.1f}%"
    if has_b:
        line += f" {byt[k]/1e6:9.1f} {byt[k]/1e3/v if v else 0:7.0f}"
    print(line)
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
if "--sweep" in sys.argv:
    keys = [k for k in tot if any(s in k for s in ("k_gemm", "k_potrf_diag", "k_panel_take"))]
    st = sum(tot[k] for k in keys); sb = sum(byt[k] for k in keys)
    print(f"dense sweep: {st:.1f} us serialised ({100*st/T:.1f}% of the step), DRAM {sb/1e6:.1f} MB per sweep")
