"""complex64 A/B of one engine option (name=value, alternated with its default to cancel
drift): DYN20 at the bench batch, RDC30 d40, VQE24 observe of 64 points.
python experiments/c64_ab.py single_blocks=0 [rounds]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, ir, sim, workloads
ctx = _lib.context()
key, val = sys.argv[1].split("=")
dflt = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
precs = sys.argv[4].split(",") if len(sys.argv) > 4 else ["c64"]
_, kd = workloads.dyn_circuit(); bd = ir.bind(kd, [])
_, kr = workloads.rdc_circuit(n=30, depth=40, every=20, seed=30200); br = ir.bind(kr, [])
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
for r in range(rounds):
    for v in (dflt, int(val)):
        ctx.set_option(key, v)
        for prec in precs:
            out = {"opt": f"{key}={v}", "prec": prec, "round": r}
            sim.sample_words(bd, 8192, 1234, precision=prec)
            sim.sample_words(bd, 8192, 1234, shot_begin=8192, precision=prec)
            out["dyn20_shots_s"] = round(8192 / (sim.last_stats()["total_ms"] / 1e3), 1)
            for _ in range(2):
                sim.run_trajectory(br, sim.RngStream.for_shot(1234, 0), precision=prec)
            out["rdc30d40_ms"] = round(sim.last_stats()["total_ms"], 1)
            sim.observe(kv, ham, pts[:8], precision=prec)
            t = time.perf_counter(); sim.observe(kv, ham, pts, precision=prec); dt = time.perf_counter() - t
            out["vqe24_points_s"] = round(64 / dt, 1)
            print(json.dumps(out), flush=True)
