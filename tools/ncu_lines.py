"""Aggregate ncu source-page (cuda,sass) stall samples per CUDA source line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
per = collections.Counter(); src = {}
cur = None
for r in rows[hdr_i + 1:]:
    if not r: continue
    if r[0] not in ("", "-") and r[0].isdigit():
        cur = int(r[0]); src[cur] = r[1][:120]
        # cuda line rows carry aggregated samples already
        try: per[cur] += int(r[si])
        except ValueError: pass
tot = sum(per.values()) or 1
for line, v in per.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{v:7d} {100*v/tot:5.1f}%  L{line}: {src[line]}")
