"""A/B of planner options on the config workloads (device time): python experiments/plan_ab.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, ir, sim, workloads
ctx = _lib.context()
_, kd = workloads.dyn_circuit(); bd = ir.bind(kd, [])
_, kr = workloads.rdc_circuit(n=30, depth=40, every=20, seed=30200); br = ir.bind(kr, [])
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
for defer in [int(x) for x in (sys.argv[1:] or ["0", "1"])]:
    ctx.set_option("defer_gates", defer)
    out = {"defer_gates": defer}
    for prec in ("c128", "c64"):
        sim.sample_words(bd, 2048, 1234, precision=prec)
        ms = []
        for r in range(3):
            sim.sample_words(bd, 2048, 1234, shot_begin=2048 * (r + 1), precision=prec)
            ms.append(sim.last_stats()["total_ms"])
        out[f"dyn20_{prec}_shots_per_s"] = 2048 / (min(ms) / 1e3)
        out[f"dyn20_{prec}_passes"] = sim.last_stats()["passes"]
        sim.run_trajectory(br, sim.RngStream.for_shot(1234, 0), precision=prec)
        sim.run_trajectory(br, sim.RngStream.for_shot(1234, 0), precision=prec)
        st = sim.last_stats()
        out[f"rdc30d40_{prec}_ms"] = st["total_ms"]
        out[f"rdc30d40_{prec}_passes"] = st["passes"]
        sim.observe(kv, ham, pts, precision=prec)
        e = sim.observe(kv, ham, pts, precision=prec)
        st = sim.last_stats()
        out[f"vqe24_{prec}_points_per_s"] = 64 / (st["total_ms"] / 1e3)
        out[f"vqe24_{prec}_pass_ms"] = st["pass_ms"]
        out[f"vqe24_{prec}_passes"] = st["passes"]
    print(json.dumps(out), flush=True)
