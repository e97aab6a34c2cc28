"""A/B of engine options (QSB option=value pairs on the command line) on DYN20 / RDC30 / VQE24:
python experiments/opt_ab.py phase_search=1 minblocks=2"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, ir, sim, workloads
ctx = _lib.context()
_, kd = workloads.dyn_circuit(); bd = ir.bind(kd, [])
_, kr = workloads.rdc_circuit(n=30, depth=40, every=20, seed=30200); br = ir.bind(kr, [])
for spec in ["base"] + sys.argv[1:]:
    if spec != "base":
        key, val = spec.split("=")
        ctx.set_option(key, int(val))
    out = {"opt": spec}
    for prec in ("c128", "c64"):
        sim.sample_words(bd, 2048, 1234, precision=prec)
        ms = []
        for r in range(2):
            sim.sample_words(bd, 2048, 1234, shot_begin=2048 * (r + 1), precision=prec)
            ms.append(sim.last_stats()["total_ms"])
        out[f"dyn20_{prec}"] = round(2048 / (min(ms) / 1e3), 1)
        for _ in range(2): sim.run_trajectory(br, sim.RngStream.for_shot(1234, 0), precision=prec)
        out[f"rdc30d40_{prec}_ms"] = round(sim.last_stats()["total_ms"], 1)
    print(json.dumps(out), flush=True)
    if spec != "base":
        from importlib import reload
        ctx.set_option(key, {"phase_search": 1, "pair_aware": 1, "minblocks": 2, "inline_phases": -1,
                             "edge_x": 1, "last_direct": 1, "fuse": 1}.get(key, 0))
