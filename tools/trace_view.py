"""Print the last dense-sweep trace (SFMCOV_SWEEP_TRACE=1 stderr) as a per-panel table."""
import sys, collections
lines = [l.split() for l in open(sys.argv[1]) if l.startswith('trace')]
calls, cur = [], []
for l in lines:
    if l[1] == 'p=0' and l[2] == 'start' and cur:
        calls.append(cur); cur = []
    cur.append(l)
calls.append(cur)
d = collections.defaultdict(dict)
for l in calls[-1]:
    d[int(l[1][2:])][l[2]] = float(l[3])
print(" p   start    take  panel   next1    rest     inv")
for p in sorted(d):
    x = d[p]
    print(f"{p:2d} {x['start']:7.3f} {x['take']:7.3f} {x['take']-x['start']:6.3f} {x.get('next1',0):7.3f} "
          f"{x.get('rest',0):7.3f} {x.get('inv',0):7.3f}")
if "--chain" in sys.argv:
    # per-launch durations on the critical stream (consecutive events of that
    # stream): mean by kind, first and second half of the panels
    chain = [l for l in calls[-1] if l[2] in ("start", "potrf", "trsm", "inner", "take", "next1")]
    np_ = max(d) + 1
    agg = collections.defaultdict(lambda: [[], []])
    for a, b in zip(chain, chain[1:]):
        if b[2] == "start":
            continue  # wait for the previous rest / inverse slot, not a launch
        agg[b[2]][int(b[1][2:]) >= np_ // 2].append((float(b[3]) - float(a[3])) * 1e3)
    print("critical-stream launch durations (us): kind, first half mean / n, second half mean / n")
    for k, (h0, h1) in agg.items():
        f = lambda v: f"{sum(v) / len(v):7.1f} / {len(v):3d}" if v else "      - /   0"
        print(f"  {k:6s} {f(h0)}   {f(h1)}")
