"""First-call (NVRTC) and steady time of RDC30 d200 under engine options:
QSB_OPTIONS=inline_phases=0 python experiments/jit_latency.py"""
import os, sys, time, json, tempfile
os.environ["QSB_JIT_CACHE"] = tempfile.mkdtemp(prefix="qsb_jit_lat_")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import ir, sim, workloads
_, k = workloads.rdc_circuit()
b = ir.bind(k, [])
out = {"options": os.environ.get("QSB_OPTIONS", "")}
for prec in ("c128", "c64"):
    t0 = time.perf_counter()
    sim.sample_words(b, 1, 1234, precision=prec)
    out[f"{prec}_first_s"] = time.perf_counter() - t0
    out[f"{prec}_first_jit_passes"] = sim.last_stats()["jit_passes"]
    out[f"{prec}_jit_ms"] = sim.last_stats()["jit_compile_ms"]
    if "jit_async=1" in out["options"]:  # wait for the background kernels
        for _ in range(120):
            sim.sample_words(b, 1, 1234, precision=prec)
            if sim.last_stats()["jit_passes"] > 0:
                break
            time.sleep(0.5)
    sim.sample_words(b, 1, 1234, precision=prec)
    out[f"{prec}_steady_ms"] = sim.last_stats()["total_ms"]
print(json.dumps(out))
