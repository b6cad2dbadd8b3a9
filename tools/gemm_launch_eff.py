"""Per-class efficiency of the dense sweep's GEMM launches: joins the stderr
log of SFMCOV_GEMM_LOG=1 (one line per launch_gemm call, in host order) with
an ncu launch list of the same process (k_gemm launches in ID order) and
prints, per launch class, launches / time / flops / TF/s (serialised,
cold-cache ncu durations: relative numbers).
usage: python tools/gemm_launch_eff.py launches.csv gemm_log.txt [calls]"""
import collections, csv, re, sys
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
dur = collections.OrderedDict()
grid = {}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum" or "k_gemm" not in r["Kernel Name"]:
        continue
    dur[int(r["ID"])] = float(r["Metric Value"].replace(",", "")) / 1e3
    grid[int(r["ID"])] = r.get("Grid Size", "")
durs = [dur[k] for k in sorted(dur)]
logs = [dict((k, int(v)) for k, v in re.findall(r"(\w+)=(-?\d+)", l)) for l in open(sys.argv[2]) if l.startswith("gemm ")]
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 1
assert len(durs) == len(logs), (len(durs), len(logs))
n = len(logs) // calls
logs, durs = logs[-n:], durs[-n:]  # the last call
def flops(g):
    t = 0.0
    if g["tri"]:
        return 2.0 * 128 * 128 * g["K"] * g["tm"] * (g["tm"] + 1) / 2
    for tj in range(g["tn"]):
        rows_ = g["tm"] - max(0, tj + g["coff"]) if g["lower"] else g["tm"]
        k = g["K"]
        if g["kfrom"] and g["b0"] >= 0 and tj >= g["b0"]:
            k -= (tj - g["b0"]) * 128
        t += 2.0 * 128 * 128 * max(k, 0) * max(rows_, 0)
    return t
def cls(g):
    if g["whole"]: return "whole-tile (in-place)"
    if g["tri"]: return f"chol trailing tri K={g['K']}"
    if g["lower"]: return f"chol panel/next cols K={g['K']} prio={g['prio']}"
    if g["kmajor"] and g["kfrom"]: return f"inv below K={g['K']}"
    if g["kmajor"] and g["alias"]: return "inv row Linv*X (alias)"
    if g["kmajor"]: return "inv in-panel rows K=128"
    return f"trsm K={g['K']}"
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for g, d in zip(logs, durs):
    a = agg[cls(g)]
    a[0] += 1; a[1] += d; a[2] += flops(g)
T = sum(a[1] for a in agg.values()); F = sum(a[2] for a in agg.values())
print(f"{'class':44s} {'n':>5s} {'ms':>8s} {'GFLOP':>9s} {'TF/s':>6s} {'time%':>6s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {a[0]:5d} {a[1]/1e3:8.3f} {a[2]/1e9:9.1f} {a[2]/a[1]/1e6:6.1f} {100*a[1]/T:5.1f}%")
print(f"{'total':44s} {sum(a[0] for a in agg.values()):5d} {T/1e3:8.3f} {F/1e9:9.1f} {F/T/1e6:6.1f}")
if "--list" in sys.argv:
    for g, d in zip(logs, durs):
        print(f"{cls(g):44s} tm={g['tm']:3d} tn={g['tn']:3d} {d:8.1f} us {flops(g)/d/1e6:6.1f} TF/s")
