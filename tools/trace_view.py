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
