"""Reducer time vs its tile run length, in a fresh process and after a large DYN20 batch
(the allocation state bench_configs leaves): python experiments/vqe_spread.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, ir, sim, workloads
ctx = _lib.context()
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
def red(lq, prec):
    ctx.set_option("expval_low_qubits", lq)
    sim.observe(kv, ham, pts, precision=prec)
    r = []
    for _ in range(3):
        sim.observe(kv, ham, pts, precision=prec)
        st = sim.last_stats()
        r.append(round(st["total_ms"] - st["pass_ms"], 1))
    return r
out = {"fresh": {f"{p}_lq{lq}": red(lq, p) for p in ("c128", "c64") for lq in (2, 3, 4)}}
_, kd = workloads.dyn_circuit()
sim.sample_words(ir.bind(kd, []), 4096, 1234)  # a 64 GiB batch, as bench_configs cfg2 leaves
out["after_dyn20"] = {f"{p}_lq{lq}": red(lq, p) for p in ("c128", "c64") for lq in (2, 3, 4)}
ctx.set_option("release_scratch", 1)
out["after_release"] = {f"{p}_lq{lq}": red(lq, p) for p in ("c128",) for lq in (2, 3)}
print(json.dumps(out))
