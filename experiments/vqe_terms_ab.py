import os, sys, json, time
sys.path.insert(0, '/root/repo')
from paper_2604_11599_b200 import _lib, sim, workloads
ctx = _lib.context()
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
for prec in ("c128", "c64"):
    for v in (32, 24, 28, 32, 24):
        ctx.set_option("expval_jit_terms", v)
        sim.observe(kv, ham, pts, precision=prec)
        ms = []
        for _ in range(5):
            sim.observe(kv, ham, pts, precision=prec); ms.append(sim.last_stats()["total_ms"])
        ms.sort()
        print(json.dumps({"prec": prec, "terms": v, "median_ms": round(ms[2], 2), "points_s": round(64 / ms[2] * 1e3, 1)}), flush=True)
