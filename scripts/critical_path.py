#!/usr/bin/env python
"""Critical path of an executed trace (offsim_execute's Chrome trace) over
the mapped task graph (build/graph_dump): which tasks and which dependency
gaps make up the executed makespan.
usage: critical_path.py graph.json trace.json"""
import collections
import json
import sys

graph = {t["name"]: t for t in json.load(open(sys.argv[1]))}
ev = {e["name"]: e for e in json.load(open(sys.argv[2]))["traceEvents"] if e.get("ph") == "X"}
byid = {t["id"]: t for t in graph.values()}
lane_prev = {}
for tid in set(e["tid"] for e in ev.values()):
    L = sorted((e for e in ev.values() if e["tid"] == tid), key=lambda e: e["ts"])
    for a, b in zip(L, L[1:]):
        lane_prev[b["name"]] = a["name"]
end = lambda n: ev[n]["ts"] + ev[n]["dur"]
cur = max(ev, key=end)
path = []
while cur:
    cands = [byid[d]["name"] for d in graph[cur]["deps"]] + ([lane_prev[cur]] if cur in lane_prev else [])
    cands = [c for c in cands if c in ev]
    pred = max(cands, key=end) if cands else None
    gap = ev[cur]["ts"] - (end(pred) if pred else 0.0)
    path.append((cur, ev[cur]["dur"], gap, "dep" if pred and pred != lane_prev.get(cur) else "lane"))
    cur = pred
path.reverse()
work = collections.Counter()
gaps = collections.Counter()
for name, dur, gap, kind in path:
    key = " ".join(name.split()[:2])
    work[key] += dur
    gaps[kind] += max(gap, 0)
print(f"makespan {max(map(end, ev)) / 1e3:.3f} ms, critical path {len(path)} tasks")
print(f"  task time {sum(work.values()) / 1e3:.3f} ms; gaps: " +
      ", ".join(f"{k} {v / 1e3:.3f} ms" for k, v in gaps.items()))
for k, v in work.most_common(12):
    print(f"    {k:24s} {v / 1e3:8.3f} ms")
