"""Reducer time vs terms per NVRTC launch: python experiments/ev_terms.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, sim, workloads
ctx = _lib.context()
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
out = {}
for prec in ("c128", "c64"):
    for nt in (16, 20, 24, 28, 32):
        ctx.set_option("expval_jit_terms", nt)
        sim.observe(kv, ham, pts, precision=prec)
        r = []
        for _ in range(3):
            e = sim.observe(kv, ham, pts, precision=prec)
            st = sim.last_stats()
            r.append(round(st["total_ms"] - st["pass_ms"], 1))
        out[f"{prec}_{nt}"] = (min(r), max(r), float(e[0]))
print(json.dumps(out))
