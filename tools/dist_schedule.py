"""Replays the 1D block-cyclic multi-GPU sweep (dist.cu) on R GPUs from the
measured per-rank work of an emulated run (the 1D-vs-2D argument).

  SFMCOV_DIST_TRACE=1 python tools/dist_schedule.py run CONFIG R 2> trace.txt
  python tools/dist_schedule.py read trace.txt [bus GB/s] [latency us]

The trace holds, for every panel p, the owner's panel factorisation f_p (its
columns' update by panel p-1, the tile chain, the hand-over; run alone on the
device) and the broadcast bytes, and for every rank r its trailing update
u_{r,p} and inverse step v_{r,p} (each alone on the device).  The replay uses
the sweep's dependencies -- f_p after the broadcast of p-1 reached the owner
and after the owner's u_{o,p-2}; broadcasts in order on one communicator
(bytes / bus bandwidth + latency); u_{r,p} after u_{r,p-1} and the broadcast of
p; v_{r,p} after v_{r,p-1} and the broadcast of p -- under two GPU models:
'serial' (each GPU runs one component at a time, panel > inverse > update
priority: pessimistic, the panel chain leaves most SMs idle) and 'overlap'
(the panel chain runs beside the updates: optimistic)."""
import collections
import sys


def parse(path):
    f, byts, u, v = {}, {}, collections.defaultdict(dict), collections.defaultdict(dict)
    R = None
    for line in open(path):
        w = line.split()
        if not w or w[0] != "dtrace":
            continue
        if w[1] == "begin":
            R = int(w[3])
            f, byts, u, v = {}, {}, collections.defaultdict(dict), collections.defaultdict(dict)  # last sweep only
        elif w[1] == "panel":
            p, o = int(w[2]), int(w[4])
            f[p] = (o, float(w[6]))
            byts[p] = int(w[8])
        elif w[1] == "update":
            p, r = int(w[2]), int(w[4])
            u[r][p] = float(w[6])
            v[r][p] = float(w[8])
    return R, f, byts, u, v


def replay(R, f, byts, u, v, bw_gbs, lat_us, overlap):
    """Discrete-event list scheduling: each GPU starts, whenever it is idle,
    its highest-priority ready component (panel > inverse step > update); the
    broadcasts share one communicator; with overlap the panel chain runs on a
    lane of its own beside the GPU's updates."""
    NP = len(f)
    items = {}  # name -> (resource, priority, duration, deps)
    for p in range(NP):
        o, fp = f[p]
        deps = [("b", p - 1)] if p > 0 else []
        if p >= 2 and p - 2 in u[o]:
            deps.append(("u", o, p - 2))
        items[("f", p)] = (("lane", o) if overlap else ("gpu", o), 0, fp, deps)
        items[("b", p)] = (("comm",), 0, byts[p] / (bw_gbs * 1e6) + lat_us * 1e-3,
                           [("f", p)] + ([("b", p - 1)] if p > 0 else []))
        for r in range(R):
            if p in v[r]:
                items[("v", r, p)] = (("gpu", r), 1, v[r][p], [("b", p)] + ([("v", r, p - 1)] if p > 0 else []))
            if p in u[r]:
                items[("u", r, p)] = (("gpu", r), 2, u[r][p], [("b", p)] + ([("u", r, p - 1)] if p > 0 else []))
    import heapq
    deps_left = {k: sum(1 for d in it[3] if d in items) for k, it in items.items()}
    users = collections.defaultdict(list)
    for k, it in items.items():
        for d in it[3]:
            if d in items:
                users[d].append(k)
    ready = collections.defaultdict(list)  # resource -> heap of (priority, panel, key)
    for k, n in deps_left.items():
        if n == 0:
            heapq.heappush(ready[items[k][0]], (items[k][1], k[-1], k))
    busy, events, done = set(), [], {}
    t = 0.0

    def dispatch():
        for res, heap in ready.items():
            if res not in busy and heap:
                _, _, k = heapq.heappop(heap)
                busy.add(res)
                heapq.heappush(events, (t + items[k][2], k))

    dispatch()
    while events:
        t, k = heapq.heappop(events)
        done[k] = t
        busy.discard(items[k][0])
        for j in users[k]:
            deps_left[j] -= 1
            if deps_left[j] == 0:
                heapq.heappush(ready[items[j][0]], (items[j][1], j[-1], j))
        dispatch()
    assert len(done) == len(items), "replay deadlock"
    return max(done.values())


if __name__ == "__main__":
    if sys.argv[1] == "run":
        sys.path.insert(0, ".")
        from paper_1808_02414_b200 import sfmcov as F
        from paper_1808_02414_b200 import synthetic as S
        rec = S.generate_config(int(sys.argv[2]))
        eng = F.Engine(0)
        eng.compute_covariance_emulated(rec, int(sys.argv[3]))
        sys.exit(0)
    R, f, byts, u, v = parse(sys.argv[2])
    bw = float(sys.argv[3]) if len(sys.argv) > 3 else 450.0
    lat = float(sys.argv[4]) if len(sys.argv) > 4 else 20.0
    work_f = sum(x[1] for x in f.values())
    work_u = sum(sum(d.values()) for d in u.values())
    work_v = sum(sum(d.values()) for d in v.values())
    per_rank = [sum(u[r].values()) + sum(v[r].values()) + sum(x[1] for x in f.values() if x[0] == r) for r in range(R)]
    total = work_f + work_u + work_v
    print(f"R = {R}, {len(f)} panels; measured work: panels {work_f:.1f} ms, updates {work_u:.1f} ms, "
          f"inverse steps {work_v:.1f} ms; total {total:.1f} ms; per rank max {max(per_rank):.1f} / mean {total / R:.1f} ms")
    print(f"broadcast: {sum(byts.values()) / 1e9:.2f} GB in total, {bw:.0f} GB/s + {lat:.0f} us per panel")
    for model in ("serial", "overlap"):
        t = replay(R, f, byts, u, v, bw, lat, model == "overlap")
        print(f"replayed sweep ({model:7s}): {t:9.1f} ms; efficiency vs total/R {total / R / t:.3f}, "
              f"vs the busiest rank {max(per_rank) / t:.3f}")
