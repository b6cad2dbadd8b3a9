"""Measured components of the dense sweep for the 1D-vs-2D multi-GPU model
(DESIGN.md §10): per-panel time from its start to its hand-over (potrf chain
+ panel trsm + inner updates: the part a 1D layout leaves on one GPU) and the
whole sweep, on one GPU, from the SFMCOV_SWEEP_TRACE=1 event trace.
usage: SFMCOV_SWEEP_TRACE=1 python tools/sweep_components.py CONFIG 2> trace.txt; python tools/sweep_components.py --read trace.txt"""
import collections
import sys

if sys.argv[1] == "--read":
    lines = [l.split() for l in open(sys.argv[2]) if l.startswith("trace")]
    calls, cur = [], []
    for l in lines:
        if l[1] == "p=0" and l[2] == "start" and cur:
            calls.append(cur)
            cur = []
        cur.append(l)
    calls.append(cur)
    d = collections.defaultdict(dict)
    for l in calls[-1]:
        d[int(l[1][2:])][l[2]] = float(l[3])
    panels = sorted(d)
    fac = [d[p]["take"] - d[p]["start"] for p in panels]
    end = max(max(v for v in d[p].values()) for p in panels)
    print(f"panels {len(panels)}; panel factorisation (start -> hand-over): sum {sum(fac):.1f} ms, "
          f"first {fac[0]:.3f} ms, median {sorted(fac)[len(fac) // 2]:.3f} ms, last {fac[-1]:.3f} ms; sweep {end:.1f} ms")
    sys.exit(0)
sys.path.insert(0, ".")
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S
rec = S.generate_config(int(sys.argv[1]))
eng = F.Engine(0)
for _ in range(2):
    eng.compute_covariance(rec)
