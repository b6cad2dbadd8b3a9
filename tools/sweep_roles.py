"""Attribute an ncu launch list of one dense sweep to the sweep's roles.

usage: sweep_roles.py launches.csv Npad [G]
Replays dense_sweep's host loop (csrc/dense.cu) to label each launch of the
LAST sweep in the list, then prints time and executed TF/s per role
(serialised, as ncu measures them)."""
import csv, sys, collections
path, Npad = sys.argv[1], int(sys.argv[2])
G = int(sys.argv[3]) if len(sys.argv) > 3 else 3
K = Npad // 128
seq = []  # (role, flops)
def gemm(role, tm, tn, k, tri=False, lower=False, row0=0):
    if tri: tiles = tm * (tm + 1) // 2
    elif lower: tiles = sum(1 for i in range(tm) for j in range(tn) if i >= j)
    else: tiles = tm * tn
    seq.append((role, 2.0 * tiles * 128 * 128 * k))
for b0 in range(0, K, G):
    g = min(G, K - b0)
    for gg in range(g):
        c = b0 + gg
        seq.append(("potrf", 0.0))
        below = K - c - 1
        if below == 0: break
        gemm("trsm", below, 1, 128)
        inner = b0 + g - c - 1
        if inner > 0: gemm("inner", below, inner, 128, lower=True)
    seq.append(("take", 0.0))
    nb0 = b0 + g; T2 = K - nb0; gn = min(T2, G)
    if T2 > gn: gemm("rest", T2 - gn, T2 - gn, g * 128, tri=True)
    if T2 > 0:
        gemm("next1", T2, 1, g * 128, lower=True)          # critical stream: the next panel's first column
        if gn > 1: gemm("next_rest", T2, gn - 1, g * 128)  # s4: its later columns
    for gg in range(g):
        r = b0 + gg
        gemm("inv_row", 1, r + 1, 128)
        later = g - gg - 1
        if later > 0: gemm("inv_panel", later, r + 1, 128)
    if T2 > 0: gemm("inv_below", T2, nb0, g * 128)
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum"]
names = [r["Kernel Name"] for r in rows]
# the sweep's launches are k_potrf_diag / k_gemm / k_panel_take; find the last run of len(seq)
dense = [i for i, n in enumerate(names) if any(k in n for k in ("k_potrf", "k_gemm", "k_panel_take"))]
sel = dense[-len(seq):]
tot = collections.defaultdict(float); fl = collections.defaultdict(float); cnt = collections.Counter()
for (role, f), i in zip(seq, sel):
    t = float(rows[i]["Metric Value"]) / 1e3  # us
    tot[role] += t; fl[role] += f; cnt[role] += 1
T = sum(tot.values())
print(f"{'role':10s} {'launches':>8s} {'total us':>9s} {'share':>6s} {'TF/s':>6s}")
for k in sorted(tot, key=lambda x: -tot[x]):
    tf = fl[k] / (tot[k] * 1e-6) / 1e12 if fl[k] else 0.0
    print(f"{k:10s} {cnt[k]:8d} {tot[k]:9.1f} {100*tot[k]/T:5.1f}% {tf:6.1f}")
print(f"serialised total {T:.1f} us, {sum(fl.values())/1e9:.1f} GFLOP executed")
