"""What a dataflow (mbarrier-per-task) warp schedule would buy over the
phase-synchronous one (wsched.Schedule): list-schedules the same tasks onto W
warps, each task starting when its producers are done (+ a sync cost), and
prints the simulated makespans side by side (cycles; `lat` cycles per op).

    python tools/dataflow_sim.py
"""
import heapq
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_06976_b200 import codegen as cg, models, wsched  # noqa: E402


def dataflow(em, warps, lat=2.0, sync=80):
    S = wsched.Schedule(em, warps)
    tasks, cost, deps = list(S.task_ops), S.cost, S.deps
    users = defaultdict(set)
    for t in tasks:
        for d in deps[t]:
            users[d].add(t)
    bl = {}

    def blev(t):
        if t not in bl:
            bl[t] = cost[t] * lat + max((blev(u) for u in users[t]), default=0)
        return bl[t]

    for t in tasks:
        blev(t)
    finish, wfree = {}, [0.0] * warps
    ready = [(-bl[t], t) for t in tasks if not deps[t]]
    heapq.heapify(ready)
    indeg = {t: len(deps[t]) for t in tasks}
    while ready:
        _, t = heapq.heappop(ready)
        est = max((finish[d] + sync for d in deps[t]), default=0)
        w = min(range(warps), key=lambda k: max(wfree[k], est))
        finish[t] = max(wfree[w], est) + cost[t] * lat
        wfree[w] = finish[t]
        for u in users[t]:
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(ready, (-bl[u], u))
    return max(finish.values()), S.critical_path() * lat + len(S.phases) * 40


if __name__ == "__main__":
    for r, w in (("chain7", 8), ("quad12", 16), ("humanoid30", 16)):
        em = cg.generate_knot(models.load(r), "gradFD", "f64")
        print(r, "dataflow %.0f vs phased %.0f" % dataflow(em, w))
    ps = wsched.variant_programs(models.load("humanoid30"), "gradFD", "f64", 10)
    print("humanoid30 variants", ["%.0f/%.0f" % dataflow(e, 8) for e in ps[:3]])
